# GPU-box script: Gaussian sketch timing, then one ncu --set full capture of the CTA-pair kernel.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/gauss_probe.py c4_1080p_gaussian 10 > gpurun_out/gauss_plain.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sketch_gaussian_tc2 -s 1 -c 1 -f -o gpurun_out/gauss_prof python tools/gauss_probe.py c4_1080p_gaussian 2 > gpurun_out/gauss_ncu.log 2>&1
echo done
