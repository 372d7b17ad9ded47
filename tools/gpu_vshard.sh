# Virtual shards (frequency-domain apply of one rank's frequency classes on 1 GPU) for the
# projected strong scaling of config 4 (E_G at G = 2, 4, 8) -- compute part only.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 2 4 8; do for r in 0 $((g-1)); do
timeout 900 python bench.py --config 4 --shard-of $g --shard-rank $r --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_v${g}_r${r}.log 2>&1
done; done
timeout 900 python bench.py --config 4 --shard-of 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/b4_v1.log 2>&1
echo done
