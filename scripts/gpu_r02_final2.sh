# Round 2 final call (after the fused eGl-QMR kernels, flat plans, plane-kernel row operands): whole GPU suite,
# smoke(), default bench line, its ncu launch list, ncu --set full of the fused tail / V~ kernel / plane-marching
# SpMM, reference arm, config 4 / 2 / 1 lines, the other global methods on config 3
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/r02_final_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_smoke.log
timeout 900 python bench.py > gpurun_out/r02_final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_bench.log
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/r02_final_bench_small.log 2>&1 || { echo "small bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_launches.csv $SMALL > gpurun_out/r02_final_ncu_launches.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qmr_tail_kernel -s 2 -c 1 -o gpurun_out/r02_final_prof_tail -f $SMALL > gpurun_out/r02_final_ncu_tail.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qmr_vt_kernel -s 2 -c 1 -o gpurun_out/r02_final_prof_vt -f $SMALL > gpurun_out/r02_final_ncu_vt.log 2>&1
echo "ncu3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_plane -s 2 -c 1 -o gpurun_out/r02_final_prof_plane -f $SMALL > gpurun_out/r02_final_ncu_plane.log 2>&1
echo "ncu4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_final_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r02_final_bench_ref.log
timeout 600 python bench.py --config 4 --no-cpu > gpurun_out/r02_final_bench_cfg4.log 2>&1
for m in gl_bicgstab egl_bicg gl_qmr gl_bicg; do timeout 600 python bench.py --config 3 --method $m --no-cpu --no-e2e > gpurun_out/r02_final_bench_cfg3_$m.log 2>&1; done
timeout 600 python bench.py --config 1 --no-cpu > gpurun_out/r02_final_bench_cfg1.log 2>&1
timeout 900 bash scripts/cfg2_methods.sh 10 > gpurun_out/r02_final_cfg2_methods.txt 2>&1
tail -n 6 gpurun_out/r02_final_all.log; tail -n 3 gpurun_out/r02_final_smoke.log; grep "^{" gpurun_out/r02_final_bench.log | cut -c1-260; grep "^{" gpurun_out/r02_final_bench_ref.log | cut -c1-260
