# Final state: whole GPU suite, smoke, default bench.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r5r_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5r_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5r_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r5r_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r5r_bench_default.log 2> gpurun_out/r5r_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5r_bench_default.err
tail -3 gpurun_out/r5r_pytest.log; tail -1 gpurun_out/r5r_smoke.log; tail -1 gpurun_out/r5r_bench_default.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/r5r_bench_default.log').read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["kernel_ms"], d["roofline"]["frac"], d["roofline"]["traffic"], d["clocks"])
P
