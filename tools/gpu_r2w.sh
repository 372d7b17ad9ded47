# far10 v5 (smem FP64 accumulators, precomputed mbarrier addresses, prefetched per-term values): parity, timings, ncu.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r2w_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2w_pytest.log
BEM_FAR_KERNEL=10 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2w_b2_far10.log 2>&1
BEM_FAR_KERNEL=10 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2w_b4_far10.log 2>&1
BEM_FAR_KERNEL=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far10" -c 1 -o gpurun_out/r2w_far10_c2 python tools/prof_apply.py --config 2 --reps 1 > gpurun_out/r2w_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2w_far10_c2.ncu-rep > gpurun_out/r2w_summary.txt 2>&1
tail -3 gpurun_out/r2w_pytest.log
echo done
