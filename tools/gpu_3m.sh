set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "h2aca_1280 or config2 or local or mask or p64" > gpurun_out/pytest_3m.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_3m.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2_3m.log 2>&1
BEM_FAR7_TTMAX=64 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2_3m_tt64.log 2>&1
echo done
