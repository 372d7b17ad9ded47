# K1 cutoff test variants (standalone kernel timers): VAR 1 (prefetched centroids, double test) vs VAR 2 (float-bit threshold), never-firing tau for both.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cutoff.py -m gpu -q > gpurun_out/r5h_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5h_pytest.log
tail -3 gpurun_out/r5h_pytest.log
for v in 1 2; do for t in 42 1e9; do
BEM_NEAR_VAR=$v BEM_NEAR_TAU=$t timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r5h_b4_v${v}_tau$t.log 2> gpurun_out/r5h_b4_v${v}_tau$t.err
done; done
BEM_NEAR_VAR=2 timeout 600 python -m pytest tests/test_gpu_cutoff.py -m gpu -q > gpurun_out/r5h_pytest_v2.log 2>&1; echo "exit $?" >> gpurun_out/r5h_pytest_v2.log
tail -3 gpurun_out/r5h_pytest_v2.log
for f in gpurun_out/r5h_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.get("work",{}).items() if k!='note'})
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
