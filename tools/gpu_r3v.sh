# HEAD validation: whole GPU suite, smoke, driver-equivalent default bench.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3v_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r3v_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3v_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r3v_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r3v_bench_default.log 2> gpurun_out/r3v_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r3v_bench_default.err
tail -3 gpurun_out/r3v_pytest.log
echo done
