# far10 with 256-entry exp / sincos tables in the B regeneration: parity (far10 tests, full-size config 4 golden), timings.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py tests/test_gpu_fullsize.py tests/test_gpu_factors.py -x -q -k "far10 or config4 or factors" > gpurun_out/r3t_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3t_pytest.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3t_b3.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3t_b4.log 2>&1
timeout 900 python bench.py --config 4 --shard-of 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3t_b4_s8.log 2>&1
tail -3 gpurun_out/r3t_pytest.log
echo done
