# ncu --set full of far10 (8 producer warps) at config 3, one launch.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far10" -c 1 -o gpurun_out/r3e_far10_c3 python tools/prof_apply.py --config 3 --reps 1 --skeleton z > gpurun_out/r3e_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r3e_far10_c3.ncu-rep > gpurun_out/r3e_summary.txt 2>&1
echo done
