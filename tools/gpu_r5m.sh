# ncu --set full of far10 under the underflow mask at config 4 and 3 (grid launch: the persistent launch's
# counter does not survive ncu's replay passes), unfused.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 4 3; do
BEM_K1_FUSE=0 BEM_FAR10_PERSIST=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"far10_kernel" -c 1 -o gpurun_out/r5m_far10_c$c python tools/prof_apply.py --config $c --reps 1 --skeleton z > gpurun_out/r5m_ncu_far10_c$c.log 2>&1
python tools/ncu_summary.py gpurun_out/r5m_far10_c$c.ncu-rep > gpurun_out/r5m_summary_far10_c$c.txt 2>&1
cat gpurun_out/r5m_summary_far10_c$c.txt
done
BEM_K1_FUSE=0 timeout 1200 ncu --set full --clock-control none -k regex:"near_kernel" -c 1 -o gpurun_out/r5m_near_c3 python tools/prof_apply.py --config 3 --reps 1 --skeleton z > gpurun_out/r5m_ncu_near_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/r5m_near_c3.ncu-rep > gpurun_out/r5m_summary_near_c3.txt 2>&1
cat gpurun_out/r5m_summary_near_c3.txt
echo done
