# Round 2: the banded SpMM — parity, then the default bench line with and without it.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_benchpath.py -q --tb=short -x > gpurun_out/r02_d.log 2>&1; echo "rc=$?" >> gpurun_out/r02_d.log
tail -n 30 gpurun_out/r02_d.log
if grep -q "rc=0" gpurun_out/r02_d.log; then
  timeout 600 python bench.py > gpurun_out/r02_d_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02_d_bench.log
  SRK_NO_BAND=1 timeout 600 python bench.py > gpurun_out/r02_d_bench_noband.log 2>&1
  python - <<'PY'
import json
for f in ("gpurun_out/r02_d_bench.log", "gpurun_out/r02_d_bench_noband.log"):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f, d["value"], d["ms_per_step"], d.get("roofline_spmm"), d["roofline"]["kernel"], d["roofline"]["frac"])
PY
fi
