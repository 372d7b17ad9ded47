# far8 distance table (DT) vs none at configs 3/4; virtual multi-rank and DT parity tests.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_comm.py tests/test_gpu_parity.py -q -x > gpurun_out/r2m_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2m_pytest.log
for dt in 0 1; do
BEM_FAR8_DT=$dt timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2m_b3_dt$dt.log 2>&1
BEM_FAR8_DT=$dt timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2m_b4_dt$dt.log 2>&1
done
echo done
