# ncu --set full of far10 at config 4 and config 3 (one launch each): stalls, pipes, DRAM traffic.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far10" -c 1 -o gpurun_out/r2y_far10_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2y_ncu4.log 2>&1
python tools/ncu_summary.py gpurun_out/r2y_far10_c4.ncu-rep > gpurun_out/r2y_summary4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far10" -c 1 -o gpurun_out/r2y_far10_c3 python tools/prof_apply.py --config 3 --reps 1 --skeleton z > gpurun_out/r2y_ncu3.log 2>&1
python tools/ncu_summary.py gpurun_out/r2y_far10_c3.ncu-rep > gpurun_out/r2y_summary3.txt 2>&1
echo done
