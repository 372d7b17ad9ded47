set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p64 or p125 or full_size or k3_variants" > gpurun_out/pt_f8grid.log 2>&1; echo "pytest exit $?" >> gpurun_out/pt_f8grid.log
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_grid.log 2>&1
timeout 900 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/b4_grid.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --replay-mode application -k regex:far8 -c 1 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/ncu_f8grid_c3.log 2>&1
echo done
