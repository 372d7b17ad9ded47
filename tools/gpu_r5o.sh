# Fused near warps taking the damped end of the K1 item list (BEM_K1_BACK=1) vs the front (0): tests, config 4 / 3.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_far10.py tests/test_gpu_step.py -m gpu -q > gpurun_out/r5o_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5o_pytest.log
tail -3 gpurun_out/r5o_pytest.log
for c in 4 3; do for k in 0 1; do
BEM_K1_BACK=$k timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5o_b${c}_back$k.log 2> gpurun_out/r5o_b${c}_back$k.err
done; done
for w in 1 2; do
BEM_K1_BACK=1 BEM_K1_WARPS=$w timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5o_b4_back1_w$w.log 2> gpurun_out/r5o_b4_back1_w$w.err
done
for f in gpurun_out/r5o_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()})
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
