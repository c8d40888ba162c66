# Round 2 session 4: BSR launch configurations (ring depth / warps / epilogue staging) — parity, sweep
mkdir -p gpurun_out
for c in 1 3 4; do SRK_BSR_CFG=$c timeout 600 python -m pytest tests/test_gpu_kernels.py -q --tb=short -k "bsr" > gpurun_out/r02u_kern_$c.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_kern_$c.log; done
BSR_TILES_ONLY=1 timeout 1200 python scripts/bsr_probe.py 32 10 > gpurun_out/r02u_bsr_cfgs.log 2>&1
tail -n 4 gpurun_out/r02u_kern_*.log; cat gpurun_out/r02u_bsr_cfgs.log
