# Round-end measurement refresh, part 2 (profiler): the launch list of a short default
# bench run and one `ncu --set full` capture of the dominant kernel (config 3's
# 6-input / 4-output update) — each only after the same command exited 0 without ncu.
mkdir -p gpurun_out
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1 || { echo "small bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:upd_kernel<double, .int.16, .bool.0, .int.6" -s 1 -c 1 -o gpurun_out/prof_upd -f $SMALL > gpurun_out/ncu_upd.log 2>&1
echo "ncu2 rc=$?"
