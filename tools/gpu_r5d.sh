# Validation of the underflow-cutoff default: whole GPU suite, smoke, driver-equivalent default bench.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r5d_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5d_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5d_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r5d_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r5d_bench_default.log 2> gpurun_out/r5d_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5d_bench_default.err
tail -4 gpurun_out/r5d_pytest.log; tail -2 gpurun_out/r5d_smoke.log; tail -1 gpurun_out/r5d_bench_default.err
echo done
