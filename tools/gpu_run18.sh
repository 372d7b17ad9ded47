set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fastmath" > gpurun_out/pytest_fm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_fm.log
BEM_NEAR_T256=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_config1 or 1280 or config2_full or p64 or p125" > gpurun_out/pytest_t256.log 2>&1; echo "exit $?" >> gpurun_out/pytest_t256.log
for v in 0 1; do BEM_NEAR_T256=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_t$v.log 2>&1; done
for v in 0 1; do BEM_NEAR_T256=$v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4h_t$v.log 2>&1; done
echo done
