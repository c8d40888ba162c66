mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_breakdown.py -m gpu -x -q --tb=short -k "flat or gl_bicg or li_bicg" > gpurun_out/r02j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_tests.log
tail -n 4 gpurun_out/r02j_tests.log
timeout 600 python bench.py --method gl_bicg --no-e2e --no-cpu > gpurun_out/r02j_bench_gl_bicg.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; tail -n 2 gpurun_out/r02j_smoke.log
timeout 600 python bench.py --no-cpu > gpurun_out/r02j_bench.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02j_bench*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:7])
PY
