# Round 2 measurement: the default bench line, its launch list, and ncu --set full captures of
# the dominant kernel (6-in / 4-out update) and the config-3 SpMM — each ncu pass only after
# the same command exited 0 without ncu. Also config 2's block methods and config 1.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench.log
timeout 600 python bench.py --config 1 --no-cpu > gpurun_out/r02_bench_cfg1.log 2>&1
timeout 600 python bench.py --config 1 --method bl_bicgstab_rq --no-cpu > gpurun_out/r02_bench_cfg1_blrq.log 2>&1
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/r02_bench_small.log 2>&1 || { echo "small bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv $SMALL > gpurun_out/r02_ncu_launches.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:upd_kernel<double, .int.16, .bool.0, .int.6" -s 1 -c 1 -o gpurun_out/r02_prof_upd -f $SMALL > gpurun_out/r02_ncu_upd.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:spmm_kernel<double, .int.16" -s 1 -c 1 -o gpurun_out/r02_prof_spmm -f $SMALL > gpurun_out/r02_ncu_spmm.log 2>&1
echo "ncu3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_kernel -c 1 -o gpurun_out/r02_prof_band -f \
  env BAND_CPLX=1 BAND_M=128 BAND_S=8 BAND_REPS=1 python scripts/band_probe.py > gpurun_out/r02_ncu_band.log 2>&1
echo "ncu4 rc=$?"
tail -n 2 gpurun_out/r02_bench.log | cut -c1-300
