# far10 v8 (compute-then-wait stage body): NB = 2 vs 3, parity for both.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for nb in 2 3; do
BEM_FAR10_NB=$nb timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3a_pytest_nb$nb.log 2>&1; echo "exit $?" >> gpurun_out/r3a_pytest_nb$nb.log
BEM_FAR10_NB=$nb timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3a_b2_nb$nb.log 2>&1
BEM_FAR10_NB=$nb timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3a_b4_nb$nb.log 2>&1
done
tail -2 gpurun_out/r3a_pytest_nb*.log
echo done
