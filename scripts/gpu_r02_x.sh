# BSR: two accumulator sets (cfg 6, 7) against the default (cfg 3) — parity and timing
mkdir -p gpurun_out
SRK_BSR_CFG=6 timeout 600 python -m pytest tests/test_gpu_kernels.py -q --tb=short -k "bsr" > gpurun_out/r02x_kern_6.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_kern_6.log
BSR_TILES_ONLY=1 BSR_CFGS=3,6,7,1,3,6 BSR_TILES=0 timeout 1200 python scripts/bsr_probe.py 32 10 > gpurun_out/r02x_bsr_cfgs.log 2>&1
tail -n 3 gpurun_out/r02x_kern_6.log; cat gpurun_out/r02x_bsr_cfgs.log
