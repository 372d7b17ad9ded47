set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cap in 220 113; do for k in 7 6; do BEM_FAR4_SMEM_KB=$cap BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_k${k}_cap$cap.log 2>&1; done; done
for cap in 220 113; do for k in 7 6; do BEM_FAR4_SMEM_KB=$cap BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_k${k}_cap$cap.log 2>&1; done; done
echo done
