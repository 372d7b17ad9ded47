set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in "BEM_FAR7_REM=1" "BEM_FAR7_REM=0" "BEM_NEAR_MINB=4" "BEM_NEAR_MINB=6" "BEM_NEAR_MINB=8" "BEM_NEAR_F=3" "BEM_NEAR_F=4"; do
  env $v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_$v.log 2>&1
done
timeout 300 python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far7" -c 1 -o gpurun_out/prof_c3far python tools/prof_apply.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
echo done
