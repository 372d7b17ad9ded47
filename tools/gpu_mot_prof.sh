set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/mot_launches.csv python tools/bench_mot.py --config 2 --N 16 > gpurun_out/mot_ncu.log 2>&1
echo done
