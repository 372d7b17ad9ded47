# Round-2 first GPU pass: factors-only skeleton, pruned K3, full-size parity, config-4 bench.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/r2a_nproc.txt; lscpu | grep "Model name" >> gpurun_out/r2a_nproc.txt; free -g >> gpurun_out/r2a_nproc.txt
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py -q > gpurun_out/r2a_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2a_pytest1.log
timeout 600 python bench.py --config 4 --skeleton z --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_b4z.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_b4f.log 2>&1
timeout 600 python bench.py --config 2 --skeleton z --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_b2z.log 2>&1
timeout 600 python bench.py --config 2 --skeleton factors --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_b2f.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s --durations=0 > gpurun_out/r2a_full.log 2>&1; echo "exit $?" >> gpurun_out/r2a_full.log
echo done
