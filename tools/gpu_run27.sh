set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
( time timeout 900 python bench.py ) > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4.log 2>&1
for c in 2 3 4; do timeout 900 python bench.py --config $c --mode h2only --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b${c}_h2o.log 2>&1; done
timeout 300 python tools/prof_apply.py --config 2 --reps 2 --time-step > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_apply.py --config 2 --reps 2 --time-step > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near|far7" -s 2 -c 2 -o gpurun_out/prof_c2_final python tools/prof_apply.py --config 2 --reps 2 > gpurun_out/ncu_full.log 2>&1
echo done
