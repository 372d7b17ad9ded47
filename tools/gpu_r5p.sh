# Config 5, one rank of 2 (round-robin shard, factors-only skeleton) under the cutoffs.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2700 python bench.py --config 5 --shard-of 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5p_b5_s2.log 2> gpurun_out/r5p_b5_s2.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/r5p_b5_s2.log').read().strip().splitlines()[-1])
print(d["ms_per_step"], d["setup_s"], d["kernel_ms"], d.get("work"), d["op"], d["skeleton"])
P
tail -3 gpurun_out/r5p_b5_s2.err
