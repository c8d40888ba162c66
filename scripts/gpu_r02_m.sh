mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_paper_table2.py tests/test_gpu_kernels.py -q --tb=short -x > gpurun_out/r02_m.log 2>&1; echo "rc=$?" >> gpurun_out/r02_m.log
timeout 600 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02_m_cfg1_blrq.log 2>&1
timeout 600 python scripts/table1_a.py r02 > gpurun_out/r02_m_table1.log 2>&1
timeout 900 python scripts/sweep_cfg5.py r02 > gpurun_out/r02_m_cfg5.log 2>&1
tail -n 15 gpurun_out/r02_m.log; grep "^{" gpurun_out/r02_m_cfg1_blrq.log | cut -c1-200; tail -4 gpurun_out/r02_m_table1.log | cut -c1-300; tail -12 gpurun_out/r02_m_cfg5.log
