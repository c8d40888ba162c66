# Round-end measurement refresh, part 1 (no profiler): GPU tests, the default bench
# line and the other configs' lines, config 2's block methods, the paper's grid.
# Outputs under gpurun_out/ (merged back); copied into profiles/ by the caller.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 600 python bench.py --config 1 --steps 200 --warmup 8 > gpurun_out/bench_cfg1.log 2>&1
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
timeout 900 bash scripts/cfg2_methods.sh 10 > gpurun_out/cfg2_methods.log 2>&1
timeout 900 python scripts/paper_grid.py r01 gpurun_out > gpurun_out/paper_grid.log 2>&1
tail -2 gpurun_out/t_gpu.log; head -c 300 gpurun_out/bench.log; echo; cat gpurun_out/cfg2_methods.log | cut -c1-60
timeout 300 python bench.py --config 1 --method bl_bicgstab_rq --steps 50 --warmup 8 > gpurun_out/bench_cfg1_blbicgstabrq.log 2>&1
timeout 300 python scripts/ilu_timing.py > gpurun_out/ilu_timing.log 2>&1
