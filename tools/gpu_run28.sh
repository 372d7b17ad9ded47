set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in 2 4 6; do BEM_H2O_FC=$v timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h2_$v.log 2>&1; done
for v in 2 3 4; do BEM_H2O_FC=$v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h4_$v.log 2>&1; done
BEM_H2O_FC=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "h2only" > gpurun_out/pytest_h2o.log 2>&1; echo "exit $?" >> gpurun_out/pytest_h2o.log
echo done
