mkdir -p gpurun_out
BAND_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_kernel -c 1 -o gpurun_out/r02_band2 python scripts/band_probe.py > gpurun_out/r02_h_ncu.log 2>&1
tail -2 gpurun_out/r02_h_ncu.log
