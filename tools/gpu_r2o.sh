# ncu captures at config 4: K4 stockham (one-shot and pipelined), K2 leaf + transfer kernels,
# far8 with the distance table; launch list and a driver-equivalent default bench.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stockham" -c 2 -o gpurun_out/r2o_k4_c4 python tools/prof_apply.py --config 4 --reps 1 --time-step --skeleton z > gpurun_out/r2o_ncu_k4.log 2>&1
BEM_FFT_PIPE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stockham" -c 1 -o gpurun_out/r2o_k4pipe_c4 python tools/prof_apply.py --config 4 --reps 1 --time-step --skeleton z > gpurun_out/r2o_ncu_k4p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"leaf_p|transfer_k" -c 26 -o gpurun_out/r2o_k2_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2o_ncu_k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8_kernel" -c 1 -o gpurun_out/r2o_far8dt_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2o_ncu_far8.log 2>&1
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2o_bench_default.log 2> gpurun_out/r2o_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2o_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2o_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2o_ncu_launch.log 2>&1
echo done
