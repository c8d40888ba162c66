# Parity tests, the default bench line, the ncu launch list of the bench command and
# one `ncu --set full` capture each of the SpMM and of the largest update kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q --tb=short > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
SMALL="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:spmm.*kernel<double, .int.16' -s 1 -c 1 -o gpurun_out/prof_spmm -f $SMALL > gpurun_out/ncu_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_spmm.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:upd_kernel<double, .int.16, .bool.0, .int.6' -s 1 -c 1 -o gpurun_out/prof_upd -f $SMALL > gpurun_out/ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_upd.log
tail -n 5 gpurun_out/t_gpu.log; tail -n 2 gpurun_out/bench.log gpurun_out/ncu_launches.log gpurun_out/ncu_spmm.log gpurun_out/ncu_upd.log
