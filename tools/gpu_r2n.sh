# Pipelined K4 (cp.async persistent Stockham) and K2 leaf kernels, far8 distance table
# (now enabled at p = 64): full GPU suite, then A/B timings.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2n_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2n_pytest.log
for pp in 0 1; do BEM_FFT_PIPE=$pp timeout 300 python tools/time_fft.py > gpurun_out/r2n_fft_pipe$pp.log 2>&1; done
for dt in 0 1; do
BEM_FAR8_DT=$dt timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_b4_dt$dt.log 2>&1
done
BEM_LEAF_PIPE=0 BEM_FFT_PIPE=0 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_b4_nopipe.log 2>&1
BEM_FAR8_DT=1 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_b3.log 2>&1
echo done
