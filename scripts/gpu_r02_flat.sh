# flat plans (Gl-BiCGStab) and lean eGl-BiCG kernels: parity tests, A/B bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_precond.py tests/test_gpu_virtual.py tests/test_gpu_breakdown.py tests/test_gpu_boundary.py tests/test_gpu_fullsize.py -m gpu -x -q --tb=short -k "flat or bicgstab or egl_bicg or benchpath or lockstep or full_solve" > gpurun_out/r02g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_tests.log
tail -n 8 gpurun_out/r02g_tests.log
for m in gl_bicgstab egl_bicg; do
  timeout 600 python bench.py --method $m --no-e2e --no-cpu > gpurun_out/r02g_bench_$m.log 2>&1
  SRK_NO_FLAT_UPDATE=1 timeout 600 python bench.py --method $m --no-e2e --no-cpu > gpurun_out/r02g_bench_${m}_generic.log 2>&1
done
timeout 600 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/r02g_bench_cfg4.log 2>&1
SRK_NO_FLAT_UPDATE=1 timeout 600 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/r02g_bench_cfg4_generic.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02g_bench_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:7])
PY
