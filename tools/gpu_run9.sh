set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python bench.py --config 5 --shard-of 8 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b5_shard8.log 2>&1; echo "exit $?" >> gpurun_out/b5_shard8.log
timeout 900 python bench.py --config 4 --shard-of 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_shard8.log 2>&1
timeout 300 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8" -c 1 -o gpurun_out/prof_c3far8 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
timeout 300 python tools/prof_apply.py --config 2 --reps 2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near|far7" -s 2 -c 2 -o gpurun_out/prof_c2b python tools/prof_apply.py --config 2 --reps 2 > gpurun_out/ncu_c2.log 2>&1
echo done
