set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "BEM_NEAR_F=3" "BEM_NEAR_F=2" "BEM_NEAR_U=1" "BEM_NEAR_F=4" "BEM_NEAR_F=4 BEM_NEAR_U=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python bench.py --config 2 --mode h2only --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s2_$tag.log 2>&1
  env $v timeout 900 python bench.py --config 4 --mode h2only --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4_$tag.log 2>&1
done
echo done
