set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q --tb=short -x > gpurun_out/t_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/t_kernels.log
timeout 1200 python -m pytest tests/test_gpu_solvers.py -q --tb=line > gpurun_out/t_solvers.log 2>&1; echo "rc=$?" >> gpurun_out/t_solvers.log
tail -5 gpurun_out/smoke.log; tail -30 gpurun_out/t_kernels.log; tail -60 gpurun_out/t_solvers.log
