# Frequency shards (one rank's share on one GPU): far10 vs far8 at config 4 / G = 2, 4, 8, and
# config 5 / G = 2 with the factors-only skeleton (far10).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 8 4 2; do
for k in 10 8; do
BEM_FAR_KERNEL=$k timeout 900 python bench.py --config 4 --shard-of $g --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3n_b4_s${g}_k$k.log 2>&1
done
done
timeout 2400 python bench.py --config 5 --shard-of 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3n_b5_s2.log 2>&1
echo done
