mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_breakdown.py -q --tb=short > gpurun_out/r02_n.log 2>&1; echo "rc=$?" >> gpurun_out/r02_n.log
timeout 900 python -m pytest tests/test_paper_table2.py -q --tb=short -k "vs_oracle" >> gpurun_out/r02_n.log 2>&1; echo "rc=$?" >> gpurun_out/r02_n.log
timeout 600 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02_n_cfg1_blrq.log 2>&1
timeout 600 python bench.py --config 1 --no-cpu > gpurun_out/r02_n_cfg1.log 2>&1
timeout 900 python scripts/sweep_cfg5.py r02 > gpurun_out/r02_n_cfg5.log 2>&1
tail -n 12 gpurun_out/r02_n.log; grep -h "^{" gpurun_out/r02_n_cfg1_blrq.log gpurun_out/r02_n_cfg1.log | cut -c1-180; head -3 gpurun_out/r02_n_cfg5.log | cut -c1-200
