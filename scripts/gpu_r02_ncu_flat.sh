# ncu --set full of a flat plan (config 4's Gl-BiCGStab P update: the third flat_kernel launch) and of the
# plane-marching SpMM's row-operand instance (config 3, Gl-BiCGStab)
mkdir -p gpurun_out
S4="python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu"
S3="python bench.py --config 3 --method gl_bicgstab --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $S4 > gpurun_out/r02l_bench_cfg4_small.log 2>&1 || { echo "cfg4 small failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flat_kernel -s 2 -c 1 -o gpurun_out/r02_final_prof_flat -f $S4 > gpurun_out/r02l_ncu_flat.log 2>&1
echo "ncu flat rc=$?"
if [ -z "$FLAT_ONLY" ]; then
timeout 600 $S3 > gpurun_out/r02l_bench_glstab_small.log 2>&1 || { echo "glstab small failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_plane -s 4 -c 1 -o gpurun_out/r02_final_prof_planerow -f $S3 > gpurun_out/r02l_ncu_planerow.log 2>&1
echo "ncu planerow rc=$?"
fi
