# Round 2: the new parity tests first, then the whole GPU suite, smoke() and the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_breakdown.py tests/test_gpu_benchpath.py -q --tb=short -x \
  > gpurun_out/r02_new.log 2>&1; echo "rc=$?" >> gpurun_out/r02_new.log
timeout 1800 python -m pytest tests -m gpu -q --tb=short \
  --deselect tests/test_gpu_virtual.py --deselect tests/test_gpu_breakdown.py --deselect tests/test_gpu_benchpath.py \
  > gpurun_out/r02_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench.log
tail -n 40 gpurun_out/r02_new.log; tail -n 15 gpurun_out/r02_all.log; tail -n 5 gpurun_out/r02_smoke.log; tail -n 3 gpurun_out/r02_bench.log
