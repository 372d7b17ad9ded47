set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --config 2 --operator K --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2_K.log 2>&1
timeout 900 python bench.py --config 4 --operator K --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_K.log 2>&1
timeout 1500 python tools/bench_solve.py --config 3 --mode h2only > gpurun_out/solve_c3_h2o.log 2>&1
timeout 1500 python tools/bench_solve.py --config 3 --dirichlet > gpurun_out/solve_c3_dir.log 2>&1
timeout 1500 python tools/bench_solve.py --config 3 > gpurun_out/solve_c3.log 2>&1
echo done
