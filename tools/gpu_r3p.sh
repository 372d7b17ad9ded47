# far10: warps past a ragged tile's end skip the A work (shards of 64 columns at G = 8).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py tests/test_gpu_comm.py -x -q > gpurun_out/r3p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3p_pytest.log
for g in 8 4; do
timeout 900 python bench.py --config 4 --shard-of $g --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3p_b4_s$g.log 2>&1
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3p_b4.log 2>&1
tail -3 gpurun_out/r3p_pytest.log
echo done
