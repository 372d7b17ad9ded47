# Checkpoint of the underflow-cutoff default (float-bit K1 test): whole GPU suite, smoke, default bench,
# reference arm, launch list of the bench command, ncu --set full of far10 and K1 (unfused) at config 4.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r5k_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r5k_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r5k_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5k_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r5k_smoke.log
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r5k_bench_default.log 2> gpurun_out/r5k_bench_default.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5k_bench_default.err
s=$(date +%s); timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r5k_bench_reference.log 2> gpurun_out/r5k_bench_reference.err; echo "rc $? wall $(( $(date +%s) - s )) s" >> gpurun_out/r5k_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r5k_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r5k_ncu_launch.log 2>&1
BEM_K1_FUSE=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"far10_kernel|near_kernel" -c 2 -o gpurun_out/r5k_k1k3_c4 python tools/prof_apply.py --config 4 --reps 1 --skeleton z > gpurun_out/r5k_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/r5k_k1k3_c4.ncu-rep > gpurun_out/r5k_summary_k1k3.txt 2>&1
tail -3 gpurun_out/r5k_pytest.log; tail -1 gpurun_out/r5k_smoke.log; tail -1 gpurun_out/r5k_bench_default.err; cat gpurun_out/r5k_summary_k1k3.txt
echo done
