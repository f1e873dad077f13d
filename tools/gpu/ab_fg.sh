# GPU-box script: A/B of library variants (lib/variants/*.so) on the full-resolution passes.
cd $GRAFT_REPO_ROOT
L=paper_1512_04205_b200/lib
cp $L/libcdmd.so /tmp/libcdmd.keep
for v in ${@:-$(ls $L/variants | sed 's/\.so$//')}; do
  cp $L/variants/$v.so $L/libcdmd.so
  { echo "=== $v"; timeout 200 python tools/fg_time.py c4_1080p_sparse 20; } >> gpurun_out/ab_fg.log 2>&1
done
cp /tmp/libcdmd.keep $L/libcdmd.so
echo done
