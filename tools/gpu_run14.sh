set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_config1 or 1280 or config2_full or h2only or fastmath" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_h2o.log 2>&1
timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_h2o.log 2>&1
timeout 300 python tools/prof_apply.py --config 2 --reps 2 --mode h2only > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near|h2o" -s 2 -c 2 -o gpurun_out/prof_c2h2o python tools/prof_apply.py --config 2 --reps 2 --mode h2only > gpurun_out/ncu_c2.log 2>&1
echo done
