# Round-2 GPU pass 4: tile-pass factors skeleton, templated Kronecker K2; config-5 shard of 2 in factors mode.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py -q -x > gpurun_out/r2d_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2d_pytest1.log
timeout 600 python bench.py --config 4 --skeleton z --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_b4z.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_b4f.log 2>&1
timeout 600 python bench.py --config 2 --skeleton z --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_b2z.log 2>&1
timeout 600 python bench.py --config 2 --skeleton factors --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_b2f.log 2>&1
timeout 300 python tools/prof_apply.py --config 3 --reps 1 --skeleton factors > gpurun_out/r2d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8|zgen_tile" -c 2 -o gpurun_out/r2d_prof_c3f python tools/prof_apply.py --config 3 --reps 1 --skeleton factors > gpurun_out/r2d_ncu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r2d_full.log 2>&1; echo "exit $?" >> gpurun_out/r2d_full.log
timeout 1500 python bench.py --config 5 --shard-of 2 --skeleton factors --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/r2d_b5s2f.log 2>&1
echo done
