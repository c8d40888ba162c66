mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_j_bench3.log 2>&1; echo "rc=$?" >> gpurun_out/r02_j_bench3.log
timeout 900 python bench.py --config 4 --steps 10 --no-cpu > gpurun_out/r02_j_bench4.log 2>&1; echo "rc=$?" >> gpurun_out/r02_j_bench4.log
python - <<'PY'
import json
for f in ("gpurun_out/r02_j_bench3.log", "gpurun_out/r02_j_bench4.log"):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f, round(d["value"]), d["median_of_5"]["value"], d["roofline"]["kernel"], round(d["roofline"]["frac"], 3),
                  {k: d["roofline_spmm"].get(k) for k in ("avg_launch_ms", "frac", "bound", "frac_of_bound", "achieved_tflops")},
                  d.get("e2e_full_solve"))
        elif "rc=" in line or "Error" in line: print(f, line.strip())
PY
