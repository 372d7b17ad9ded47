set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/plain4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"near|far8" -c 2 -o gpurun_out/prof_c4 python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
timeout 300 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near|far8" -c 2 -o gpurun_out/prof_c3 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
echo done
