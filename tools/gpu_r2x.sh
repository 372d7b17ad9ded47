# far10 as the default K3: the whole GPU suite, smoke, default bench (config 4), config 2/3 lines.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2x_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2x_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2x_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2x_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r2x_bench_default.log 2> gpurun_out/r2x_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2x_bench_default.err
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2x_b2.log 2>&1
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2x_b3.log 2>&1
tail -5 gpurun_out/r2x_pytest.log
echo done
