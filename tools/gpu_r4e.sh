# K1 fusion diagnostics: items done by the fused warps, and the per-kernel launch times (ncu, one pass).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_K1_FUSE_STATS=1 timeout 600 python tools/prof_apply.py --config 3 --reps 2 > gpurun_out/r4e_stats_c3.log 2>&1
BEM_K1_FUSE_STATS=1 timeout 600 python tools/prof_apply.py --config 4 --reps 2 > gpurun_out/r4e_stats_c4.log 2>&1
for fu in 1 0; do
BEM_K1_FUSE=$fu timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"far10|near|xmax|seg_red" --csv python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/r4e_ncu_c3_f$fu.csv 2>gpurun_out/r4e_ncu_c3_f$fu.err
done
grep -h "K1 fused" gpurun_out/r4e_stats_c*.log
echo done
