cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 600 python -m pytest tests -m gpu -q -rf -k "partition or lanczos or smoke" > gpurun_out/lz3_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lz3_smoke.log 2>&1
echo "smoke rc $?" >> gpurun_out/lz3_smoke.log
echo done
