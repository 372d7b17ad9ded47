# far10 leftover-column FP64 work moved before the stage's buffer wait (loads overlap the slice regeneration).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r4j_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4j_pytest.log
for fu in 1 0; do
BEM_K1_FUSE=$fu timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4j_b4_f$fu.log 2>&1
BEM_K1_FUSE=$fu timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4j_b3_f$fu.log 2>&1
done
tail -2 gpurun_out/r4j_pytest.log
for f in gpurun_out/r4j_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"coupling": [0-9.]*' $f|head -1) $(grep -o '"near": [0-9.]*' $f | head -1)"; done
echo done
