set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for k in 8 7; do BEM_FAR_KERNEL=$k timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_k$k.log 2>&1; done
for k in 8 7; do BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_k$k.log 2>&1; done
BEM_FAR_KERNEL=8 BEM_FAR8_KC=64 BEM_FAR4_SMEM_KB=220 timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_k8_kc64.log 2>&1
for k in 8 7; do BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_k$k.log 2>&1; done
echo done
