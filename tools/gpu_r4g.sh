# Fused K1 warps per persistent far10 CTA (BEM_K1_WARPS = 1, 2, 3) at configs 4 and 3.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for w in 1 2 3; do
BEM_K1_WARPS=$w BEM_K1_FUSE_STATS=1 timeout 600 python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/r4g_stats_c4_w$w.log 2>&1
BEM_K1_WARPS=$w timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4g_b4_w$w.log 2>&1
BEM_K1_WARPS=$w timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4g_b3_w$w.log 2>&1
done
grep -h "K1 fused" gpurun_out/r4g_stats_c4_w*.log
for f in gpurun_out/r4g_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
echo done
