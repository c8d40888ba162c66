mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_virtual.py -q --tb=short > gpurun_out/r02_k.log 2>&1; echo "rc=$?" >> gpurun_out/r02_k.log
SRK_NO_HALO_OVERLAP=1 timeout 900 python -m pytest tests/test_gpu_virtual.py -q --tb=short -k "full_solve" >> gpurun_out/r02_k.log 2>&1; echo "rc=$?" >> gpurun_out/r02_k.log
tail -n 30 gpurun_out/r02_k.log
