mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_virtual.py -q --tb=short -k bsr > gpurun_out/r02_l.log 2>&1; echo "rc=$?" >> gpurun_out/r02_l.log
tail -n 30 gpurun_out/r02_l.log
