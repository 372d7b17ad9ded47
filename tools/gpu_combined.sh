# GPU check of the combined mode (NEXT-4): parity tests + config 2/3 bench lines + K1m ncu capture.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_combined.py -q -x > gpurun_out/pytest_combined.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_combined.log
timeout 600 python bench.py --config 2 --mode combined --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b2_comb.log 2>&1
timeout 900 python bench.py --config 3 --mode combined --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b3_comb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nearm -c 1 -o gpurun_out/nearm_c2 -f python tools/prof_apply.py --config 2 --mode combined --reps 1 > gpurun_out/ncu_nearm.log 2>&1
echo done
