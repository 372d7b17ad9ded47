set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in 1 0; do BEM_OVERLAP=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/o2_$v.log 2>&1; done
for v in 1 0; do BEM_OVERLAP=$v timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/o2h_$v.log 2>&1; done
for v in 1 0; do BEM_OVERLAP=$v timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o4_$v.log 2>&1; done
for v in 1 0; do BEM_OVERLAP=$v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o4h_$v.log 2>&1; done
echo done
