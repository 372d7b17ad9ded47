set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench_default.log 2>&1
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_reference.log 2>&1
timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2_h2o.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4.log 2>&1
echo done
