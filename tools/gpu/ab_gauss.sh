# GPU-box script: A/B of library variants (lib/variants/*.so) on the Gaussian and SRFT sketches.
cd $GRAFT_REPO_ROOT
L=paper_1512_04205_b200/lib
cp $L/libcdmd.so /tmp/libcdmd.keep
for v in ${@:-$(ls $L/variants | sed 's/\.so$//')}; do
  cp $L/variants/$v.so $L/libcdmd.so
  { echo "=== $v $(nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader)"
    timeout 200 python tools/gauss_probe.py c4_1080p_gaussian 10
    timeout 200 python tools/gauss_probe.py c3_720x480_rademacher 10 gaussian
    timeout 200 python tools/gauss_probe.py c4_1080p_gaussian 6 srft
  } >> gpurun_out/ab_gauss.log 2>&1
done
cp /tmp/libcdmd.keep $L/libcdmd.so
echo done
