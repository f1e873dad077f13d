# GPU-box script: A/B of library variants (lib/variants/*.so) on the 3x3 median pass.
cd $GRAFT_REPO_ROOT
L=paper_1512_04205_b200/lib
cp $L/libcdmd.so /tmp/libcdmd.keep
for v in ${@:-$(ls $L/variants | sed 's/\.so$//')}; do
  cp $L/variants/$v.so $L/libcdmd.so
  { echo "=== $v"; timeout 100 python tools/median3_time.py; } >> gpurun_out/ab_med.log 2>&1
done
cp /tmp/libcdmd.keep $L/libcdmd.so
echo done
