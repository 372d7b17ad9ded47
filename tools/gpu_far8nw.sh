set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR8_NW=6 BEM_FAR7_M3=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p64 or full_size or p125" > gpurun_out/pytest_f8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_f8.log
BEM_FAR8_NW=6 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_nw6.log 2>&1
BEM_FAR8_NW=6 BEM_FAR7_M3=1 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_nw6m3.log 2>&1
echo done
