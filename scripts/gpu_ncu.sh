# ncu captures of the two dominant kernels of the eGl-QMR config-3 step.
mkdir -p gpurun_out
SMALL="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1; echo "plain rc=$?" >> gpurun_out/bench_small.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:spmm_kernel<double, 16' -s 1 -c 1 -o gpurun_out/prof_spmm -f $SMALL > gpurun_out/ncu_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_spmm.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:upd_kernel<double, 16' -s 5 -c 1 -o gpurun_out/prof_upd -f $SMALL > gpurun_out/ncu_upd.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_upd.log
tail -2 gpurun_out/bench_small.log gpurun_out/ncu_spmm.log gpurun_out/ncu_upd.log
