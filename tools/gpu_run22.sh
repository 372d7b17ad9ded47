set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "p64 or p125" > gpurun_out/pytest_f9.log 2>&1; echo "exit $?" >> gpurun_out/pytest_f9.log
for k in 9 8; do BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_k$k.log 2>&1; done
for k in 9 8; do BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_k$k.log 2>&1; done
echo done
