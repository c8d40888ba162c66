# Round 2 session 3: plane-marching SpMM (7-point operators) + ILUTP — parity, timing, ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_band.py -q --tb=short -x > gpurun_out/r02p_band.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_band.log
timeout 600 python -m pytest tests/test_gpu_precond.py -q --tb=short -k ilutp > gpurun_out/r02p_ilutp.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_ilutp.log
for pl in 1 0; do SRK_BAND_PLANE=$pl timeout 300 python scripts/band_probe.py > gpurun_out/r02p_probe_$pl.log 2>&1; done
BAND_CPLX=1 BAND_M=128 BAND_S=8 timeout 300 python scripts/band_probe.py > gpurun_out/r02p_probe_c128.log 2>&1
BAND_CPLX=1 BAND_M=128 BAND_S=8 SRK_BAND_PLANE=0 timeout 300 python scripts/band_probe.py > gpurun_out/r02p_probe_c128_0.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/r02p_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_bench.log
BAND_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_plane --launch-skip 3 -c 1 -o gpurun_out/r02p_plane python scripts/band_probe.py > gpurun_out/r02p_ncu.log 2>&1
tail -n 4 gpurun_out/r02p_band.log gpurun_out/r02p_ilutp.log; cat gpurun_out/r02p_probe_*.log; grep "^{" gpurun_out/r02p_bench.log | cut -c1-400; tail -n 3 gpurun_out/r02p_ncu.log
