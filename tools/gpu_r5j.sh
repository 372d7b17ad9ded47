# K1 fused into far10 vs separate K1 (side stream) under the cutoffs, config 4 and 3, graph replay.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 4 3; do for f in 0 1; do
BEM_K1_FUSE=$f timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5j_b${c}_f$f.log 2> gpurun_out/r5j_b${c}_f$f.err
done; done
BEM_K1_FUSE=1 BEM_K1_WARPS=2 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5j_b4_f1_w2.log 2> gpurun_out/r5j_b4_f1_w2.err
for f in gpurun_out/r5j_b*.log; do python - "$f" <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"],1), {k:round(v,1) for k,v in d["kernel_ms"].items()}, d["timing"][:90])
except Exception as e:
    print(sys.argv[1], "ERR", e)
P
done
