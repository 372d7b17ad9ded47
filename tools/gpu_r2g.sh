# Driver-equivalent bench runs (default N=1 line and the reference arm), wall-clock timed.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench_default.log 2> gpurun_out/r2g_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2g_bench_default.err
s=$(date +%s); timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2g_bench_reference.log 2> gpurun_out/r2g_bench_reference.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2g_bench_reference.err
echo done
