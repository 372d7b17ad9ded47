# K4 at L = 513: register-resident two-pass kernel (k513) vs the generic Stockham kernel.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "transforms or time_step" > gpurun_out/r3f_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3f_pytest.log
timeout 600 python -m pytest tests/test_gpu_step.py -q >> gpurun_out/r3f_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3f_pytest.log
for v in 1 0; do BEM_FFT_513=$v timeout 300 python tools/time_fft.py > gpurun_out/r3f_fft_$v.log 2>&1; done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3f_b4.log 2>&1
tail -3 gpurun_out/r3f_pytest.log
echo done
