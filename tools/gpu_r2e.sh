# Round-2 GPU pass 5: CTA-cooperative Z regeneration (right-looking substitutions), paired-output prime DFT stages.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py -q -x > gpurun_out/r2e_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2e_pytest1.log
timeout 600 python bench.py --config 4 --skeleton z --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_b4z.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_b4f.log 2>&1
timeout 600 python bench.py --config 2 --skeleton z --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_b2z.log 2>&1
timeout 600 python bench.py --config 2 --skeleton factors --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_b2f.log 2>&1
timeout 300 python tools/time_fft.py > gpurun_out/r2e_fft.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r2e_full.log 2>&1; echo "exit $?" >> gpurun_out/r2e_full.log
echo done
