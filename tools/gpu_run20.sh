set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_NEAR_STAGED=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_config1 or 1280 or config2_full or p64 or edge or local or mask" > gpurun_out/pytest_staged.log 2>&1; echo "exit $?" >> gpurun_out/pytest_staged.log
for v in 0 1; do BEM_NEAR_STAGED=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_s$v.log 2>&1; done
for v in 0 1; do BEM_NEAR_STAGED=$v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4h_s$v.log 2>&1; done
echo done
