set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
BEM_NEAR_LEAN=1 timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_lean.log 2>&1
for i in 1 2; do timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_h2o_$i.log 2>&1; done
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4.log 2>&1
BEM_NEAR_LEAN=1 timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_lean.log 2>&1
timeout 300 python tools/prof_apply.py --config 2 --reps 2 --mode h2only --time-step > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_h2o.csv python tools/prof_apply.py --config 2 --reps 2 --mode h2only --time-step > gpurun_out/ncu_launch.log 2>&1
echo done
