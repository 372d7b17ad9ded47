set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_apply.py --config 2 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"aca_kernel" -c 1 -o gpurun_out/prof_aca python tools/prof_apply.py --config 2 --reps 1 > gpurun_out/ncu_aca.log 2>&1
echo done
