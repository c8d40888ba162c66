# One GPU call: parity tests, the default bench line, an ncu launch list and one
# `ncu --set full` capture of the dominant kernel (B200_PROFILING.md recipe).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q --tb=short -p no:randomly > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
SMALL="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:spmm_kernel<double, 16' -s 1 -c 1 -o gpurun_out/prof_spmm $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
tail -25 gpurun_out/t_gpu.log; tail -3 gpurun_out/bench.log; tail -3 gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
