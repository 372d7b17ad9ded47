# Round-2 evidence pass: everything the driver runs at round end, plus ncu captures at config 4.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2f_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2f_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2f_smoke.log
/usr/bin/time -v timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench_default.log 2> gpurun_out/r2f_bench_default.err
/usr/bin/time -v timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2f_bench_reference.log 2> gpurun_out/r2f_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2f_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8_kernel" -c 1 -o gpurun_out/r2f_far8_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2f_ncu_far8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near_kernel|up_leaf_d|down_leaf_d|up_transfer_k|down_transfer_k|gather" -c 8 -o gpurun_out/r2f_k1k2_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2f_ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham" -c 2 -o gpurun_out/r2f_k4_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z --time-step > gpurun_out/r2f_ncu_k4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"zgen_tile|far7_kernel" -c 2 -o gpurun_out/r2f_zgen_c2 python tools/prof_apply.py --config 2 --reps 1 --skeleton factors > gpurun_out/r2f_ncu_zgen.log 2>&1
echo done
