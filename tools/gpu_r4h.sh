# Validation of the fused K1 / persistent far10 default: whole GPU suite, smoke, driver-equivalent default
# bench, and the ncu launch list of a short run of the same bench command.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r4h_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r4h_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4h_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r4h_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r4h_bench_default.log 2> gpurun_out/r4h_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r4h_bench_default.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4h_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4h_ncu_launch.log 2>&1
tail -3 gpurun_out/r4h_pytest.log
echo done
