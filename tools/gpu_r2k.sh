# K4 NC sweep; compute-sanitizer racecheck of every hot kernel.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for nc in 1 2 4 8; do BEM_FFT_NC=$nc timeout 300 python tools/time_fft.py > gpurun_out/r2k_fft_nc$nc.log 2>&1; done
bash tools/gpu_sanitize.sh racecheck
echo done
