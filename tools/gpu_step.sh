set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -q -x > gpurun_out/pytest_step.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_step.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/b4.log 2>&1
echo done
