# Multi-rank flow on one GPU: 2 ranks (gloo process group), fused peer transpose vs all-to-all.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for t in peer a2a; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$([ $t = peer ] && echo 1 || echo 2) bench.py --gpus 2 --dist-backend gloo --transpose $t --config 2 --steps 3 --warmup 3 > gpurun_out/b2_2rank_$t.log 2>&1; echo "exit $?" >> gpurun_out/b2_2rank_$t.log
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
echo done
