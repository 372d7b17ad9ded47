# Config-3 CQM solve (BASELINE config 3: GMRES per frequency to 1e-8) with far10, and the double
# layer / combined-mode bench lines at config 3.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python tools/bench_solve.py --config 3 > gpurun_out/r3r_solve_c3.log 2>&1
timeout 900 python bench.py --config 3 --operator K --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3r_b3_dl.log 2>&1
timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3r_b4_h2o.log 2>&1
echo done
