# Gl-QMR (V~, W~) flat plan: parity tests, A/B bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_precond.py tests/test_gpu_virtual.py tests/test_gpu_breakdown.py -m gpu -x -q --tb=short -k "flat or fused or qmr" > gpurun_out/r02k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_tests.log
tail -n 4 gpurun_out/r02k_tests.log
timeout 600 python bench.py --method gl_qmr --no-e2e --no-cpu > gpurun_out/r02k_bench_gl_qmr.log 2>&1
SRK_NO_FLAT_UPDATE=1 timeout 600 python bench.py --method gl_qmr --no-e2e --no-cpu > gpurun_out/r02k_bench_gl_qmr_generic.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02k_bench*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:7])
PY
