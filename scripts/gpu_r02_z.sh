# Round 2 final: whole GPU suite, smoke(), default bench line, its ncu launch list, config 1 / 4 lines
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/r02z_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_smoke.log
timeout 900 python bench.py > gpurun_out/r02z_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_bench.log
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/r02z_bench_small.log 2>&1 || { echo "small bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02z_launches.csv $SMALL > gpurun_out/r02z_ncu_launches.log 2>&1
echo "ncu1 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02z_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_bench_ref.log
tail -n 6 gpurun_out/r02z_all.log; tail -n 3 gpurun_out/r02z_smoke.log; grep "^{" gpurun_out/r02z_bench.log | cut -c1-260; grep "^{" gpurun_out/r02z_bench_ref.log | cut -c1-260
