# Round-robin frequency shards under the cutoffs: whole GPU suite again (shard / comm / peer tests), per-rank cost of
# config-4 shards (G = 2, 4, 8; first and last rank), config-3 solve timing, config 5 rank 0 of 8.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r5l_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5l_pytest.log
tail -3 gpurun_out/r5l_pytest.log
for gr in "2 0" "2 1" "4 0" "4 3" "8 0" "8 3" "8 7"; do set -- $gr
timeout 900 python bench.py --config 4 --shard-of $1 --shard-rank $2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5l_b4_s$1_r$2.log 2> gpurun_out/r5l_b4_s$1_r$2.err
done
timeout 1500 python tools/bench_solve.py --config 3 > gpurun_out/r5l_solve_c3.log 2>&1
timeout 1800 python bench.py --config 5 --shard-of 8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5l_b5_s8_r0.log 2> gpurun_out/r5l_b5_s8_r0.err
for f in gpurun_out/r5l_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.get("work",{}).items() if k!='note'})
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
tail -5 gpurun_out/r5l_solve_c3.log
echo done
