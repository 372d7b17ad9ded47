# Underflow cutoffs (K1 class cutoff, far10 (block, tile) mask): new tests, the far10 / factors / fused
# suites, then config 4 and 3 with the cutoffs on (default) and off.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_far10.py tests/test_gpu_factors.py -m gpu -q -x > gpurun_out/r5a_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5a_pytest.log
tail -5 gpurun_out/r5a_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5a_b4_on.log 2> gpurun_out/r5a_b4_on.err
BEM_NEAR_TAU=0 BEM_FAR_SKIP_LOG2=0 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5a_b4_off.log 2> gpurun_out/r5a_b4_off.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5a_b3_on.log 2> gpurun_out/r5a_b3_on.err
BEM_NEAR_TAU=0 BEM_FAR_SKIP_LOG2=0 timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5a_b3_off.log 2> gpurun_out/r5a_b3_off.err
for f in gpurun_out/r5a_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["ms_per_step"], d["kernel_ms"], d.get("work"), d["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
echo done
