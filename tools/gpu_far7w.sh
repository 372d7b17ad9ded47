set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BEM_FAR7_NW=16 BEM_FAR7_M3=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "h2aca_1280 or config2 or local or mask or solve_h2aca or edge" > gpurun_out/pytest_w.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_w.log
for v in "8 0" "16 0" "16 1"; do set -- $v
BEM_FAR7_NW=$1 BEM_FAR7_M3=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b2_nw$1_m$2.log 2>&1
done
echo done
