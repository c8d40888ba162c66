# Parity tests + the default bench line (no profiler).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q --tb=short > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -n 30 gpurun_out/t_gpu.log; tail -n 2 gpurun_out/bench.log
