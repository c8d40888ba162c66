# Round 2: boundary options (shadow, preprocess, eps, vector_ops) and a quick regression of f3/f4.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_f3f4.py -q --tb=short > gpurun_out/r02_c.log 2>&1; echo "rc=$?" >> gpurun_out/r02_c.log
tail -n 60 gpurun_out/r02_c.log
