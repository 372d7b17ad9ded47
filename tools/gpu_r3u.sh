# far10 role split (BEM_FAR10_PW=17: 8 A warps + 8 B warps) vs the default (8 combined warps).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR10_PW=17 timeout 900 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3u_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3u_pytest.log
for pw in 17 8; do
BEM_FAR10_PW=$pw timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3u_b3_pw$pw.log 2>&1
BEM_FAR10_PW=$pw timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3u_b4_pw$pw.log 2>&1
done
tail -3 gpurun_out/r3u_pytest.log
echo done
