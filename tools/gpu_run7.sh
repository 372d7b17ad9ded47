set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in "BEM_NEAR_F=3" "BEM_NEAR_MINB=4" "BEM_NEAR_MINB=2" "BEM_NEAR_F=2"; do
  env $v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_$v.log 2>&1
done
for c in 3 4; do for cap in 113 220; do BEM_FAR4_SMEM_KB=$cap timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b${c}_cap$cap.log 2>&1; done; done
timeout 900 python tools/bench_solve.py --config 1 --check-freqs 4 > gpurun_out/solve_c1.log 2>&1
timeout 1500 python tools/bench_solve.py --config 3 --check-freqs 3 > gpurun_out/solve_c3.log 2>&1
echo done
