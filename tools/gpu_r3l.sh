# far10 (unsigned A) with 16 vs 8 producer warps at configs 3 and 4.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for pw in 16 8; do
BEM_FAR10_PW=$pw timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3l_b3_pw$pw.log 2>&1
BEM_FAR10_PW=$pw timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3l_b4_pw$pw.log 2>&1
done
BEM_FAR10_PW=16 timeout 600 python -m pytest tests/test_gpu_far10.py -x -q > gpurun_out/r3l_pytest_pw16.log 2>&1; echo "exit $?" >> gpurun_out/r3l_pytest_pw16.log
echo done
