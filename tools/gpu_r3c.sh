# far10 CTA pairs (cta_group::2): parity (pair and single), timings.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3c_pytest_pair.log 2>&1; echo "exit $?" >> gpurun_out/r3c_pytest_pair.log
BEM_FAR10_PAIR=0 timeout 600 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3c_pytest_single.log 2>&1; echo "exit $?" >> gpurun_out/r3c_pytest_single.log
for pr in 1 0; do
BEM_FAR10_PAIR=$pr timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3c_b3_p$pr.log 2>&1
BEM_FAR10_PAIR=$pr timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3c_b4_p$pr.log 2>&1
done
tail -2 gpurun_out/r3c_pytest_*.log
echo done
