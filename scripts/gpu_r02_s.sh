# Round 2 session 4: SELL + team-kernel regression tests, config 4 / config 1 / config 2 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sell.py -q --tb=short > gpurun_out/r02s_sell.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_sell.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q --tb=short -x > gpurun_out/r02s_kern.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_kern.log
timeout 900 python bench.py --config 4 --no-cpu --no-e2e --steps 10 > gpurun_out/r02s_bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_bench_cfg4.log
timeout 300 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02s_bench_cfg1_blrq.log 2>&1
timeout 300 python bench.py --config 1 --no-cpu > gpurun_out/r02s_bench_cfg1.log 2>&1
timeout 900 bash scripts/cfg2_methods.sh 10 > gpurun_out/r02s_cfg2_methods.txt 2>&1
tail -n 6 gpurun_out/r02s_sell.log gpurun_out/r02s_kern.log; for f in cfg4 cfg1_blrq cfg1; do grep "^{" gpurun_out/r02s_bench_$f.log | cut -c1-260; done; cat gpurun_out/r02s_cfg2_methods.txt
