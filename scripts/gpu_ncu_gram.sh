# ncu --set full of the DMMA Gram kernel (s = 64), after the same command ran clean
mkdir -p gpurun_out
timeout 300 python scripts/gram_probe.py > gpurun_out/gram_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gram_mma_kernel" -c 1 \
  -o gpurun_out/prof_gram -f python scripts/gram_probe.py > gpurun_out/ncu_gram.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gram.log
tail -n 3 gpurun_out/ncu_gram.log
