cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
CDMD_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline_parity_small or philox or gaussian_table or spixel_rows or sparse_rows" > gpurun_out/lz5_pytest_$i.log 2>&1
done
echo done
