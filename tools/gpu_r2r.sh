# ncu capture of far10 v1 at config 2 (one launch) for stall reasons / pipe usage.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR_KERNEL=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far10" -c 1 -o gpurun_out/r2r_far10_c2 python tools/prof_apply.py --config 2 --reps 1 > gpurun_out/r2r_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2r_far10_c2.ncu-rep > gpurun_out/r2r_summary.txt 2>&1
echo done
