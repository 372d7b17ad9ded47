set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4.log 2>&1
timeout 1500 python bench.py --config 5 --shard-of 8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b5.log 2>&1
echo done
