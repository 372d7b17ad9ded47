# Round-2 third GPU pass: Kronecker/DMMA K2, ILP zgen, hoisted real-slice branch; ncu of far8 at config 3.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py -q -x > gpurun_out/r2c_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2c_pytest1.log
timeout 600 python bench.py --config 4 --skeleton z --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_b4z.log 2>&1
timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_b4f.log 2>&1
BEM_LIB_PATH=$PWD/exp/libbem_noinl.so timeout 600 python bench.py --config 4 --skeleton factors --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_b4f_noinl.log 2>&1
timeout 600 python bench.py --config 2 --skeleton z --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_b2z.log 2>&1
timeout 600 python bench.py --config 2 --skeleton factors --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_b2f.log 2>&1
timeout 300 python tools/prof_apply.py --config 3 --reps 1 --skeleton z > gpurun_out/r2c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far8|up_leaf_d|down_leaf_d|up_transfer_k|stockham" -c 6 -o gpurun_out/r2c_prof_c3 python tools/prof_apply.py --config 3 --reps 1 --skeleton z > gpurun_out/r2c_ncu.log 2>&1
echo done
