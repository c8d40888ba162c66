# Round 2 session 4: BSR-12 M = 24 / K = 12 tensor-core form and SELL-32-sigma — parity, timing, DRAM bytes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q --tb=short -x -k "bsr or config5 or spmm_matches or fused or lattice" > gpurun_out/r02r_kern.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_kern.log
timeout 900 python -m pytest tests/test_gpu_sell.py -q --tb=short > gpurun_out/r02r_sell.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_sell.log
timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_solvers.py -q --tb=short -k "bsr or lattice or cfg4" > gpurun_out/r02r_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_bsr.log
timeout 900 python scripts/sweep_cfg5.py r02 > gpurun_out/r02r_sweep.log 2>&1
SRK_NO_SELL=1 timeout 900 python scripts/sweep_cfg5.py r02_nosell > gpurun_out/r02r_sweep_nosell.log 2>&1
cp profiles/r02_cfg5_sweep.json profiles/r02_nosell_cfg5_sweep.json gpurun_out/ 2>/dev/null
timeout 600 python scripts/table1_a.py r02 > gpurun_out/r02r_table1.log 2>&1; cp profiles/r02_table1_a.json gpurun_out/ 2>/dev/null
timeout 1200 python scripts/bsr_probe.py 32 10 > gpurun_out/r02r_bsr_probe.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:bsr12 -c 20 --csv --log-file gpurun_out/r02r_bsr_ncu.csv python scripts/bsr_probe.py 32 1 > gpurun_out/r02r_bsr_ncu.log 2>&1
tail -n 5 gpurun_out/r02r_kern.log gpurun_out/r02r_sell.log gpurun_out/r02r_bsr.log; cat gpurun_out/r02r_bsr_probe.log; grep -E "^\{" gpurun_out/r02r_sweep.log | cut -c1-200; grep -E "^\{" gpurun_out/r02r_sweep_nosell.log | cut -c1-120; tail -n 8 gpurun_out/r02r_table1.log; grep bsr12 gpurun_out/r02r_bsr_ncu.csv | cut -c1-300
