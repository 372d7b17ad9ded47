set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3.log 2>&1
BEM_FAR_KERNEL=6 timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_k6.log 2>&1
timeout 300 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far7|near" -c 2 -o gpurun_out/prof_c3 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
echo done
