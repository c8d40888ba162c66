# plane-marching SpMM with row operands, hoisted n-vector loads: parity tests, A/B bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_band.py tests/test_gpu_benchpath.py tests/test_gpu_solvers.py tests/test_gpu_kernels.py -m gpu -x -q --tb=short -k "plane or band or benchpath or lockstep or bicgstab or spmm" > gpurun_out/r02h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_tests.log
tail -n 8 gpurun_out/r02h_tests.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/r02h_bench_egl_qmr.log 2>&1
timeout 600 python bench.py --method egl_bicg --no-e2e --no-cpu > gpurun_out/r02h_bench_egl_bicg.log 2>&1
timeout 600 python bench.py --method gl_bicgstab --no-e2e --no-cpu > gpurun_out/r02h_bench_gl_bicgstab.log 2>&1
SRK_NO_PLANE_ROWS=1 timeout 600 python bench.py --method gl_bicgstab --no-e2e --no-cpu > gpurun_out/r02h_bench_gl_bicgstab_norows.log 2>&1
timeout 600 python bench.py --config 2 --method gl_bicgstab --no-e2e --no-cpu > gpurun_out/r02h_bench_cfg2_gl_bicgstab.log 2>&1
SRK_NO_PLANE_ROWS=1 timeout 600 python bench.py --config 2 --method gl_bicgstab --no-e2e --no-cpu > gpurun_out/r02h_bench_cfg2_gl_bicgstab_norows.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02h_bench_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], round(d["value"], 1), round(d["ms_per_step"], 3), [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3)) for k in d["iteration"]["kernels"]][:7])
PY
