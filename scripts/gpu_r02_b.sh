# Round 2: f3 / f4 parity, the breakdown and bench-path tests, and the tests that failed in r02_tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_f3f4.py tests/test_gpu_breakdown.py tests/test_gpu_benchpath.py \
  "tests/test_gpu_solvers.py::test_lattice_lockstep_and_solve" "tests/test_gpu_solvers.py::test_full_solve" \
  -q --tb=short > gpurun_out/r02_b.log 2>&1; echo "rc=$?" >> gpurun_out/r02_b.log
tail -n 60 gpurun_out/r02_b.log
