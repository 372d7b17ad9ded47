# K1 early exit (source leaves by distance + suffix distances): K1-relevant suites, config 4 / 3 / 2 benches.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_far10.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r5e_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5e_pytest.log
tail -15 gpurun_out/r5e_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5e_b4_on.log 2> gpurun_out/r5e_b4_on.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5e_b3_on.log 2> gpurun_out/r5e_b3_on.err
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5e_b2_on.log 2> gpurun_out/r5e_b2_on.err
for f in gpurun_out/r5e_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.get("work",{}).items() if k!='note'}, round(d["roofline"]["frac"],3), d["per_kernel_roofline"]["kernels"]["near"]["frac"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
echo done
