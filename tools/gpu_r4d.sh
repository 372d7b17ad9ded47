# K1 fused into far10 (3 near-field warps per far10 CTA + a tail kernel): parity and config 3/4 step times,
# fused (default) vs BEM_K1_FUSE=0.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_far10.py tests/test_gpu_step.py -x -q > gpurun_out/r4d_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4d_pytest.log
for fu in 1 0; do
BEM_K1_FUSE=$fu timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4d_b4_f$fu.log 2>&1
BEM_K1_FUSE=$fu timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4d_b3_f$fu.log 2>&1
done
tail -3 gpurun_out/r4d_pytest.log
for f in gpurun_out/r4d_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o 'eager step [0-9.]*' $f) $(grep -o '"coupling": [0-9.]*' $f|head -1) $(grep -o '"near": [0-9.]*' $f | head -1)"; done
echo done
