set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:aca_kernel -c 1 -o gpurun_out/aca_c4 -f python tools/prof_apply.py --config 4 --reps 0 > gpurun_out/ncu_aca.log 2>&1
echo done
