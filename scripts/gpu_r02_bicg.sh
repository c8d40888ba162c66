# Gl-BiCG flat plans + restructured A/B tests: parity, A/B bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_precond.py tests/test_gpu_virtual.py tests/test_gpu_breakdown.py -m gpu -x -q --tb=short -k "benchpath or flat or fused or gl_bicg or lockstep" > gpurun_out/r02i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02i_tests.log
tail -n 8 gpurun_out/r02i_tests.log
timeout 600 python bench.py --method gl_bicg --no-e2e --no-cpu > gpurun_out/r02i_bench_gl_bicg.log 2>&1
SRK_NO_FLAT_UPDATE=1 timeout 600 python bench.py --method gl_bicg --no-e2e --no-cpu > gpurun_out/r02i_bench_gl_bicg_generic.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02i_bench_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:7])
PY
