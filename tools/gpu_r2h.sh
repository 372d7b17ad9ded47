# far9 (warp-specialised K3) correctness and speed.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py -q -x > gpurun_out/r2h_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2h_pytest1.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h_b4.log 2>&1
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h_b3.log 2>&1
BEM_FAR_KERNEL=8 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h_b3_far8.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h_b4f.log 2>&1
echo done
