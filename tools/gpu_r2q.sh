# far10 (K3 on INT8 tensor cores): parity tests, then config 2 / 4 timings against far8.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py tests/test_gpu_tc.py -x -q > gpurun_out/r2q_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2q_pytest.log
BEM_FAR_KERNEL=10 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2q_b2_far10.log 2>&1
BEM_FAR_KERNEL=10 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2q_b4_far10.log 2>&1
tail -3 gpurun_out/r2q_pytest.log
echo done
