# Persistent far10 (BEM_FAR10_PERSIST, named barriers for the coupling warps) with the fused K1 warps
# (BEM_K1_FUSE): parity, fused-item counts, config 3/4 step times for the four combinations.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py tests/test_gpu_step.py -x -q > gpurun_out/r4f_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4f_pytest.log
BEM_K1_FUSE_STATS=1 timeout 600 python tools/prof_apply.py --config 4 --reps 2 > gpurun_out/r4f_stats_c4.log 2>&1
for v in "1 1" "1 0" "0 1" "0 0"; do set -- $v
BEM_FAR10_PERSIST=$1 BEM_K1_FUSE=$2 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4f_b4_p$1_f$2.log 2>&1
BEM_FAR10_PERSIST=$1 BEM_K1_FUSE=$2 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4f_b3_p$1_f$2.log 2>&1
done
tail -3 gpurun_out/r4f_pytest.log
grep -h "K1 fused" gpurun_out/r4f_stats_c4.log
for f in gpurun_out/r4f_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o 'eager step [0-9.]*' $f) $(grep -o '"coupling": [0-9.]*' $f|head -1) $(grep -o '"near": [0-9.]*' $f | head -1)"; done
echo done
