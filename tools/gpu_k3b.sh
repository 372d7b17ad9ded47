set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "h2aca or p64 or p125 or config2 or mask or local or full_size" > gpurun_out/pytest_k3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k3.log
timeout 600 python bench.py --config 2 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b2.log 2>&1
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3.log 2>&1
echo done
