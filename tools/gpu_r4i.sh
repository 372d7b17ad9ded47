# ncu --set full of the persistent far10 at config 3, with (default) and without the fused K1 warps.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:far10 -c 1 -o gpurun_out/r4i_far10_fused_c3 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/r4i_ncu_fused.log 2>&1
BEM_K1_FUSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:far10 -c 1 -o gpurun_out/r4i_far10_plain_c3 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/r4i_ncu_plain.log 2>&1
ls -la gpurun_out/
echo done
