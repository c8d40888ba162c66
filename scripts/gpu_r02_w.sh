# Round 2 session 4 (final measurement): update-kernel parity after the partial ring, config 2 lines,
# the default bench line, its ncu launch list, and ncu --set full of the dominant update, the
# plane-marching SpMM and the BSR product (each ncu pass only after the same command exited 0 without ncu)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_f3f4.py -q --tb=short -x -k "update or block or bl_ or cfg2 or cplx" > gpurun_out/r02w_upd.log 2>&1; echo "rc=$?" >> gpurun_out/r02w_upd.log
timeout 900 bash scripts/cfg2_methods.sh 10 > gpurun_out/r02w_cfg2_methods.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02w_bench.log
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/r02w_bench_small.log 2>&1 || { echo "small bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02w_launches.csv $SMALL > gpurun_out/r02w_ncu_launches.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:upd_kernel<double, .int.16, .bool.0, .int.6" -s 1 -c 1 -o gpurun_out/r02w_prof_upd -f $SMALL > gpurun_out/r02w_ncu_upd.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_plane -s 1 -c 1 -o gpurun_out/r02w_prof_plane -f $SMALL > gpurun_out/r02w_ncu_plane.log 2>&1
echo "ncu3 rc=$?"
BSR_TILES_ONLY=1 BSR_CFGS=3 BSR_TILES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsr12_kernel2 --launch-skip 2 -c 1 -o gpurun_out/r02w_prof_bsr -f python scripts/bsr_probe.py 32 1 > gpurun_out/r02w_ncu_bsr.log 2>&1
echo "ncu4 rc=$?"
tail -n 4 gpurun_out/r02w_upd.log; cat gpurun_out/r02w_cfg2_methods.txt | cut -c1-220; grep "^{" gpurun_out/r02w_bench.log | cut -c1-300
