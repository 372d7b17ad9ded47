# K1 cutoff with the float-bit test (single variant, float-bit suffix distances): suites and benches.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_far10.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r5i_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5i_pytest.log
tail -4 gpurun_out/r5i_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5i_b4_on.log 2> gpurun_out/r5i_b4_on.err
BEM_NEAR_TAU=1e9 timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r5i_b4_tau1e9.log 2> gpurun_out/r5i_b4_tau1e9.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5i_b3_on.log 2> gpurun_out/r5i_b3_on.err
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5i_b2_on.log 2> gpurun_out/r5i_b2_on.err
for f in gpurun_out/r5i_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.get("work",{}).items() if k!='note'}, d["per_kernel_roofline"]["kernels"]["near"]["frac"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
