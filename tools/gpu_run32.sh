set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
echo done
