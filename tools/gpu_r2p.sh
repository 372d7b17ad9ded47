# Re-entry check of HEAD: full GPU suite, smoke, default (driver-equivalent) bench, launch list.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2p_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2p_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2p_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r2p_bench_default.log 2> gpurun_out/r2p_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r2p_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2p_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2p_ncu_launch.log 2>&1
echo done
