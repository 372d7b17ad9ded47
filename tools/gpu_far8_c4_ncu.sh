set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --replay-mode application -k regex:far8 -c 1 -o gpurun_out/far8_c4 -f python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/ncu_far8_c4.log 2>&1
echo done
