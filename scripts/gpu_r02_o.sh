# Round 2 (session 3): state of HEAD — whole GPU suite, smoke(), default bench line, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02o_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02o_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_smoke.log
timeout 600 python bench.py > gpurun_out/r02o_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_bench.log
timeout 600 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02o_cfg1_blrq.log 2>&1
grep -E "passed|failed|error" gpurun_out/r02o_all.log | tail -5; grep -E "^(FAILED|ERROR)" gpurun_out/r02o_all.log | head -20; tail -n 3 gpurun_out/r02o_smoke.log; grep "^{" gpurun_out/r02o_bench.log | cut -c1-300; grep "^{" gpurun_out/r02o_cfg1_blrq.log | cut -c1-200
