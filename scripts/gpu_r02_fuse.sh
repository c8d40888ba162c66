# fused QMR tail / vector fusion: parity tests, A/B bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_precond.py tests/test_gpu_virtual.py tests/test_gpu_breakdown.py tests/test_gpu_boundary.py -m gpu -x -q --tb=short -k "qmr or benchpath or QMR" > gpurun_out/r02f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_tests.log
tail -n 8 gpurun_out/r02f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_smoke.log; tail -n 3 gpurun_out/r02f_smoke.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/r02f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_bench.log
SRK_NO_QMR_VEC_FUSE=1 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/r02f_bench_novec.log 2>&1
python - <<'PY'
import json
for f in ("r02f_bench.log", "r02f_bench_novec.log"):
    for l in open("gpurun_out/" + f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:8])
PY
