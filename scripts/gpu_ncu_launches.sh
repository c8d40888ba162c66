# ncu launch list (gpu__time_duration per launch) of a short bench run; run after
# the same command has exited 0 without ncu (scripts/gpu_tests_bench.sh).
mkdir -p gpurun_out
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
tail -n 3 gpurun_out/ncu_launches.log
