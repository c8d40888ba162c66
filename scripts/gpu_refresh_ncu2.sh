# Round-end refresh, part 3: config 1 / 4 bench lines with their documented step
# counts, and ncu --set full captures of config 2's tensor-core kernels (the block
# update and the per-warp Gram), each after the same command exited 0 without ncu.
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 --steps 200 --warmup 8 > gpurun_out/bench_cfg1.log 2>&1
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
C2="python bench.py --config 2 --method bl_bicg_rq --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $C2 > gpurun_out/bench_c2.log 2>&1 || { echo "c2 bench failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:upd_mma_kernel" -s 3 -c 1 -o gpurun_out/prof_updmma -f $C2 > gpurun_out/ncu_updmma.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:gram_warp_kernel" -s 2 -c 1 -o gpurun_out/prof_gramwarp -f $C2 > gpurun_out/ncu_gramwarp.log 2>&1
echo "ncu2 rc=$?"
