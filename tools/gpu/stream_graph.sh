cd $GRAFT_REPO_ROOT
timeout 600 python tools/stream_graph_probe.py 10 40 > gpurun_out/sg.log 2>&1
timeout 600 python tools/stream_graph_probe.py 16 64 >> gpurun_out/sg.log 2>&1
