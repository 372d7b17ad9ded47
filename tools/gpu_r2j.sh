# 3M default, register prime radix in K4: tests + bench + fft timing.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py -q -x > gpurun_out/r2j_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2j_pytest1.log
timeout 300 python tools/time_fft.py > gpurun_out/r2j_fft.log 2>&1
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j_b4.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j_b4f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham" -c 2 -o gpurun_out/r2j_k4_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z --time-step > gpurun_out/r2j_ncu_k4.log 2>&1
echo done
