# K1 launched right after K3 (BEM_K1_LATE=1: K3 on the highest-priority stream, graph nodes keep
# their priorities) vs the default fork: step time (graph replay) at configs 4 and 3; parity.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_K1_LATE=1 timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_far10.py -x -q > gpurun_out/r3m_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3m_pytest.log
for kl in 1 0; do
BEM_K1_LATE=$kl timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3m_b4_kl$kl.log 2>&1
BEM_K1_LATE=$kl timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3m_b3_kl$kl.log 2>&1
done
tail -3 gpurun_out/r3m_pytest.log
echo done
