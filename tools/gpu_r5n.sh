# Final validation: whole GPU suite, bounds-checked library on the cutoff / far10 / factors / parity / comm suites,
# smoke, default bench, reference arm, launch list of the bench command.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r5n_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5n_pytest.log
BEM_LIB_PATH=$PWD/paper_2006_05186_b200/libbem_checked.so timeout 1500 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_far10.py tests/test_gpu_factors.py tests/test_gpu_parity.py tests/test_gpu_comm.py tests/test_gpu_step.py -q > gpurun_out/r5n_checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5n_checked_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5n_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r5n_smoke.log
s=$(date +%s); timeout 1800 python bench.py > gpurun_out/r5n_bench_default.log 2> gpurun_out/r5n_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5n_bench_default.err
s=$(date +%s); timeout 1800 python bench.py --impl reference > gpurun_out/r5n_bench_reference.log 2> gpurun_out/r5n_bench_reference.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5n_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r5n_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r5n_ncu_launch.log 2>&1
tail -3 gpurun_out/r5n_pytest.log; tail -3 gpurun_out/r5n_checked_pytest.log; tail -1 gpurun_out/r5n_smoke.log; tail -1 gpurun_out/r5n_bench_default.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/r5n_bench_default.log').read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["kernel_ms"], d["work"]["k1_evals_run_frac"], d["work"]["k3_rank_cols_run_frac"], d["roofline"]["frac"], d["clocks"])
P
echo done
