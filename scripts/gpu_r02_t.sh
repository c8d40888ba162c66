# Round 2 session 4: block-row visiting order (BSR), flat view of awkward-width scalar updates — parity, timing, DRAM bytes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sell.py tests/test_gpu_kernels.py -q --tb=short -k "sell or team or bsr or update or gram" > gpurun_out/r02t_kern.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_kern.log
timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_virtual.py tests/test_gpu_boundary.py -q --tb=short -x > gpurun_out/r02t_solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_solvers.log
BSR_TILES_ONLY=1 timeout 900 python scripts/bsr_probe.py 32 10 > gpurun_out/r02t_bsr_tiles.log 2>&1
BSR_TILES_ONLY=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bsr12 -c 40 --csv --log-file gpurun_out/r02t_bsr_ncu.csv python scripts/bsr_probe.py 32 1 > gpurun_out/r02t_bsr_ncu.log 2>&1
timeout 900 python bench.py --config 4 --no-cpu --no-e2e --steps 10 > gpurun_out/r02t_bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_bench_cfg4.log
tail -n 6 gpurun_out/r02t_kern.log gpurun_out/r02t_solvers.log; cat gpurun_out/r02t_bsr_tiles.log; grep "^{" gpurun_out/r02t_bench_cfg4.log | cut -c1-200
python - <<'P'
import csv
rows = [r for r in csv.reader(open("gpurun_out/r02t_bsr_ncu.csv")) if len(r) > 14 and r[0].isdigit()]
by = {}
for r in rows: by.setdefault(int(r[0]), {})[r[12]] = float(r[14].replace(",", ""))
for k in sorted(by): print(k, {m: round(v / 1e9, 2) if "bytes" in m else round(v / 1e6, 3) for m, v in by[k].items()})
P
