set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/peaks.py > gpurun_out/peaks.json 2>&1
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "exit $?" >> gpurun_out/bench_c$c.log; done
timeout 600 python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/prof_apply.py --config 4 --reps 1 > gpurun_out/ncu_launch4.log 2>&1
echo done
