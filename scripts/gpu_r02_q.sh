# Round 2 session 4: state check after the container was re-created — the whole GPU suite (no -x, every
# failure listed), smoke(), the default bench line, and the GPU's eGl-QMR counts at 96^3 / 128^3 / 256^3
# (the count-ensemble study, scripts/oracle_counts.py m128 ...).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02q_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02q_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02q_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02q_smoke.log
timeout 900 python bench.py > gpurun_out/r02q_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02q_bench.log
timeout 600 python scripts/gpu_counts.py 96 128 256 > gpurun_out/r02q_counts.log 2>&1
tail -n 30 gpurun_out/r02q_all.log; tail -n 3 gpurun_out/r02q_smoke.log; grep "^{" gpurun_out/r02q_bench.log | cut -c1-300; cat gpurun_out/r02q_counts.log
