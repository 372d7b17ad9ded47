# far8 3M (16-row mu chunks) vs 4M: correctness and speed at configs 3 and 4.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p64_multi_tile or p125" > gpurun_out/r2i_pytest1.log 2>&1; echo "exit $?" >> gpurun_out/r2i_pytest1.log
for m3 in 0 1; do
BEM_FAR8_M3=$m3 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_b3_m3$m3.log 2>&1
BEM_FAR8_M3=$m3 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_b4_m3$m3.log 2>&1
done
echo done
