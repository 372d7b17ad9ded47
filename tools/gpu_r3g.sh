# K2 transfer tile width sweep (BEM_K2_TF) at config 4: per-kernel ms from the bench's profiler pass.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tf in 0 4 8 16; do
BEM_K2_TF=$tf timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3g_b4_tf$tf.log 2>&1
done
echo done
