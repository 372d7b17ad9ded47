# far10 CTA pairs with 8 producer warps (one slice entry per thread per CTA): parity and timing.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR10_PAIR=1 timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3q_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3q_pytest.log
for pr in 1 0; do
BEM_FAR10_PAIR=$pr timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3q_b3_p$pr.log 2>&1
BEM_FAR10_PAIR=$pr timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3q_b4_p$pr.log 2>&1
done
tail -3 gpurun_out/r3q_pytest.log
echo done
