# One `ncu --set full` capture of one kernel of the bench step:
#   bash scripts/gpu_ncu_full.sh spmm 'regex:spmm.*kernel<double, .int.16'
#   bash scripts/gpu_ncu_full.sh upd  'regex:upd_kernel<double, .int.16, .bool.0, .int.6'
mkdir -p gpurun_out
NAME=$1
KREGEX=$2
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$KREGEX" -s 1 -c 1 \
  -o gpurun_out/prof_$NAME -f $SMALL > gpurun_out/ncu_$NAME.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$NAME.log
tail -n 3 gpurun_out/ncu_$NAME.log
