# GPU check of the time-domain path (NEXT-2): parity tests + MoT vs frequency solve timings.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mot.py -q -x > gpurun_out/pytest_mot.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mot.log
timeout 600 python tools/bench_mot.py --config 2 --N 16 > gpurun_out/mot_c2_n16.log 2>&1
timeout 600 python tools/bench_mot.py --config 2 --N 32 > gpurun_out/mot_c2_n32.log 2>&1
timeout 900 python tools/bench_mot.py --config 2 --N 128 > gpurun_out/mot_c2_n128.log 2>&1
echo done
