# far10: 16 vs 8 producer warps (BEM_FAR10_PW), parity for both, timings.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for pw in 16 8; do
BEM_FAR10_PW=$pw timeout 600 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3d_pytest_pw$pw.log 2>&1; echo "exit $?" >> gpurun_out/r3d_pytest_pw$pw.log
BEM_FAR10_PW=$pw timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3d_b3_pw$pw.log 2>&1
BEM_FAR10_PW=$pw timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3d_b4_pw$pw.log 2>&1
done
tail -2 gpurun_out/r3d_pytest_*.log
echo done
