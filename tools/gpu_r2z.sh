# far10 v7 (3-stage pipeline with the third A stage in shared memory, one mbarrier arrival per warp).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r2z_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2z_pytest.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_b2.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_b4.log 2>&1
tail -3 gpurun_out/r2z_pytest.log
echo done
