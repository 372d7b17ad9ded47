# K2 leaf kernels: sub-tiles per CTA sweep (BEM_LEAF_SUB) at config 4 with TF = 4 transfers.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for sub in 8 4 2 1; do
BEM_LEAF_SUB=$sub timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3h_b4_sub$sub.log 2>&1
done
echo done
