# GPU-box script: ONE compute-sanitizer tool (argument 1: memcheck | racecheck | synccheck |
# initcheck) over the small cases of tools/sanitize_cases.py, after a plain run exits 0.
cd $GRAFT_REPO_ROOT
TOOL=${1:-memcheck}
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 &&
timeout 1500 compute-sanitizer --tool $TOOL --kernel-name kns=cdmd --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_$TOOL.log 2>&1
echo "sanitizer exit $?" >> gpurun_out/san_$TOOL.log
echo done
