# K1 co-scheduled with K3: BEM_K1_LATE (K3 on a high-priority stream, K1 launched after it on the
# lowest-priority stream) x BEM_K1_NW (warps per K1 CTA: 4 default, 1 fits next to a far10 CTA).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_K1_LATE=1 BEM_K1_NW=1 timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_far10.py -x -q > gpurun_out/r4a_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4a_pytest.log
for v in "0 4" "1 1" "0 1" "1 4"; do set -- $v
BEM_K1_LATE=$1 BEM_K1_NW=$2 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4a_b4_l$1_nw$2.log 2>&1
done
BEM_K1_LATE=1 BEM_K1_NW=1 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4a_b3_l1_nw1.log 2>&1
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4a_b3_l0_nw4.log 2>&1
tail -3 gpurun_out/r4a_pytest.log
for f in gpurun_out/r4a_b*.log; do echo $f; grep -o '"ms_per_step": [0-9.]*' $f; done
echo done
