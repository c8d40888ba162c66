# Round 2 session 4: whole GPU suite, smoke(), the bench lines of configs 3 (default) / 4 / 1 / 2
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02v_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02v_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_smoke.log
timeout 900 python bench.py > gpurun_out/r02v_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_bench.log
timeout 900 python bench.py --config 4 --no-cpu > gpurun_out/r02v_bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_bench_cfg4.log
timeout 300 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02v_bench_cfg1_blrq.log 2>&1
timeout 300 python bench.py --config 1 --no-cpu > gpurun_out/r02v_bench_cfg1.log 2>&1
timeout 900 bash scripts/cfg2_methods.sh 10 > gpurun_out/r02v_cfg2_methods.txt 2>&1
tail -n 12 gpurun_out/r02v_all.log; tail -n 3 gpurun_out/r02v_smoke.log; for f in "" _cfg4 _cfg1_blrq _cfg1; do grep "^{" gpurun_out/r02v_bench$f.log | cut -c1-230; done; cat gpurun_out/r02v_cfg2_methods.txt | cut -c1-200
