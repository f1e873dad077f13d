cd $GRAFT_REPO_ROOT
timeout 300 python tools/fg_time.py c4_1080p_sparse 30 > gpurun_out/fg_time.log 2>&1
timeout 300 python tools/fg_time.py c4_1080p_sparse 30 >> gpurun_out/fg_time.log 2>&1
