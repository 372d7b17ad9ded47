# As r4b, with K1 and far10 both asking for the maximum shared-memory carveout (an SM's carveout is
# one setting for all resident CTAs).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "1 1 1" "0 1 1" "0 0 4" "1 1 4"; do set -- $v
BEM_FAR10_PERSIST=$1 BEM_K1_LATE=$2 BEM_K1_NW=$3 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4c_b4_p$1_l$2_nw$3.log 2>&1
done
for f in gpurun_out/r4c_b*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o 'eager step [0-9.]*' $f) $(grep -o '"coupling": [0-9.]*' $f|head -1) $(grep -o '"near": [0-9.]*' $f | head -1)"; done
echo done
