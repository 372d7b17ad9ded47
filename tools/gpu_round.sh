# Canonical GPU-box run (gpurun -- 'bash tools/gpu_round.sh'): tests, smoke, the driver's
# bench line, the reference arm, the other configs, the plain-H2 ablation, solves, and an
# ncu launch list + full capture of K1/K3 at config 2.  Outputs under gpurun_out/.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
python tools/peaks.py > gpurun_out/peaks.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4.log 2>&1
for c in 2 3 4; do timeout 900 python bench.py --config $c --mode h2only --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b${c}_h2o.log 2>&1; done
timeout 1800 python bench.py --config 5 --shard-of 8 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b5_shard8.log 2>&1
timeout 1500 python tools/bench_solve.py --config 3 > gpurun_out/solve_c3.log 2>&1
timeout 600 python bench.py --config 2 --mode combined --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2_comb.log 2>&1
timeout 600 python tools/bench_mot.py --config 2 --N 16 > gpurun_out/mot_c2_n16.log 2>&1
timeout 300 python tools/prof_apply.py --config 2 --reps 2 --time-step > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_apply.py --config 2 --reps 2 --time-step > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near|far7" -s 2 -c 2 -o gpurun_out/prof_c2 python tools/prof_apply.py --config 2 --reps 2 > gpurun_out/ncu_full.log 2>&1
echo done
