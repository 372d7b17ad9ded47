# Plain-H2 (K3') underflow cutoff: cutoff + parity suites, config 4 / 3 h2only benches on / off.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r5q_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5q_pytest.log
tail -4 gpurun_out/r5q_pytest.log
for c in 4 3; do
timeout 900 python bench.py --config $c --mode h2only --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5q_b${c}_h2o_on.log 2> gpurun_out/r5q_b${c}_h2o_on.err
done
BEM_NEAR_TAU=0 timeout 900 python bench.py --config 4 --mode h2only --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5q_b4_h2o_off.log 2> gpurun_out/r5q_b4_h2o_off.err
for f in gpurun_out/r5q_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, d["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
