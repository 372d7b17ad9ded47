set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b2_ov.log 2>&1
BEM_OVERLAP=0 timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b2_noov.log 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_ov.log 2>&1
timeout 600 python bench.py --config 2 --mode h2only --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2h_ov.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config2 or h2aca_1280 or local or mask or solve" > gpurun_out/pytest_ov.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ov.log
echo done
