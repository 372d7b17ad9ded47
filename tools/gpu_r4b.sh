# Persistent far10 (BEM_FAR10_PERSIST=1: one CTA per SM taking work items from a counter) so that
# K1 launched after it (BEM_K1_LATE=1) can fill the SM slots far10 leaves free (BEM_K1_NW=1: one-warp
# CTAs, 2: one-warp CTAs of 2 classes at <= 88 registers).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR10_PERSIST=1 BEM_K1_LATE=1 BEM_K1_NW=1 timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_far10.py -x -q > gpurun_out/r4b_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4b_pytest.log
BEM_FAR10_PERSIST=1 BEM_K1_LATE=1 BEM_K1_NW=2 timeout 900 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/r4b_pytest2.log 2>&1; echo "exit $?" >> gpurun_out/r4b_pytest2.log
for v in "1 0 4" "1 1 1" "1 1 2" "0 0 2" "0 0 4"; do set -- $v
BEM_FAR10_PERSIST=$1 BEM_K1_LATE=$2 BEM_K1_NW=$3 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4b_b4_p$1_l$2_nw$3.log 2>&1
done
tail -3 gpurun_out/r4b_pytest*.log
for f in gpurun_out/r4b_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o 'eager step [0-9.]*' $f) $(grep -o '"coupling": [0-9.]*' $f) $(grep -o '"near": [0-9.]*' $f)"; done
echo done
