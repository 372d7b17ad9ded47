set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for kb in 0 120; do
BEM_FAR_SMEM_MIN_KB=$kb timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2_smem$kb.log 2>&1
BEM_FAR_SMEM_MIN_KB=$kb BEM_OVERLAP=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2_smem${kb}_noov.log 2>&1
BEM_FAR_SMEM_MIN_KB=$kb timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_smem$kb.log 2>&1
done
echo done
