mkdir -p gpurun_out
python scripts/band_probe.py > gpurun_out/r02_e_probe.txt 2>&1
SRK_NO_BAND=1 python scripts/band_probe.py >> gpurun_out/r02_e_probe.txt 2>&1
BAND_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_kernel -c 2 -o gpurun_out/r02_band python scripts/band_probe.py > gpurun_out/r02_e_ncu.log 2>&1
cat gpurun_out/r02_e_probe.txt; tail -3 gpurun_out/r02_e_ncu.log
