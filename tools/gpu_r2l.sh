# Bounds-checked library on the GPU tests (memory-safety evidence; compute-sanitizer is not
# available on this pool), then the default bench and the config-4 K3 capture with 3M far8.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_LIB_PATH=$PWD/paper_2006_05186_b200/libbem_checked.so timeout 600 python tools/sanitize_case.py > gpurun_out/r2l_checked_cases.log 2>&1; echo "exit $?" >> gpurun_out/r2l_checked_cases.log
BEM_LIB_PATH=$PWD/paper_2006_05186_b200/libbem_checked.so timeout 1500 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py tests/test_gpu_combined.py tests/test_gpu_mot.py tests/test_gpu_step.py -q > gpurun_out/r2l_checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2l_checked_pytest.log
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench_default.log 2> gpurun_out/r2l_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2l_bench_default.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8_kernel" -c 1 -o gpurun_out/r2l_far8m3_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r2l_ncu_far8.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2l_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2l_ncu_launch.log 2>&1
echo done
