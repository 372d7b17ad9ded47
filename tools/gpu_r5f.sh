# K1 code-path check: cutoff compiled in but never firing (tau = 1e9) vs off vs on, config 4, per-kernel timers only.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 1e9 0 42; do
BEM_NEAR_TAU=$t timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r5f_b4_tau$t.log 2> gpurun_out/r5f_b4_tau$t.err
done
for f in gpurun_out/r5f_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.get("work",{}).items() if k!='note'})
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
