set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in 4 5 6; do
  BEM_NEAR_F=$v timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f2_$v.log 2>&1
  BEM_NEAR_F=$v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f4_$v.log 2>&1
done
BEM_NEAR_F=5 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_config1 or 1280 or config2_full" > gpurun_out/pytest_f5.log 2>&1; echo "exit $?" >> gpurun_out/pytest_f5.log
echo done
