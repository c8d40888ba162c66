# Round-end refresh, part 3: ncu --set full captures of config 2's tensor-core block
# update and config 1's single-CTA iteration kernel, each after the same command exited
# 0 without ncu.
mkdir -p gpurun_out
C2="python bench.py --config 2 --method bl_bicg_rq --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $C2 > gpurun_out/bench_c2.log 2>&1 || { echo "c2 bench failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:upd_mma_kernel" -s 3 -c 1 -o gpurun_out/prof_updmma -f $C2 > gpurun_out/ncu_updmma.log 2>&1
echo "ncu1 rc=$?"
C1="python bench.py --config 1 --steps 20 --warmup 8 --no-e2e --no-cpu"
timeout 600 $C1 > gpurun_out/bench_c1.log 2>&1 || { echo "c1 bench failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:egl_bicg_small" -s 4 -c 1 -o gpurun_out/prof_small -f $C1 > gpurun_out/ncu_small.log 2>&1
echo "ncu2 rc=$?"
