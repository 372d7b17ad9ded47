set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR7_M3=1 BEM_FAR7_TTMAX=64 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p64 or full_size" > gpurun_out/pytest_f8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_f8.log
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_base.log 2>&1
BEM_FAR7_TTMAX=64 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_tt64.log 2>&1
BEM_FAR7_M3=1 BEM_FAR7_TTMAX=64 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_m3.log 2>&1
echo done
