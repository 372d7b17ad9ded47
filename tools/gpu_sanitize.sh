# compute-sanitizer on every hot kernel (tools/sanitize_case.py; 1280-panel cases).  One tool per call:
#   gpurun -- 'bash tools/gpu_sanitize.sh racecheck'   /   ... memcheck / synccheck / initcheck
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tool=${1:-racecheck}
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_case.py > gpurun_out/r2_sanitize_$tool.log 2>&1
echo "exit $?" >> gpurun_out/r2_sanitize_$tool.log
tail -5 gpurun_out/r2_sanitize_$tool.log
