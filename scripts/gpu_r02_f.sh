mkdir -p gpurun_out
: > gpurun_out/r02_f_sweep.txt
for tr in 16 32 64; do for d in 2 3 4 6 8; do
  sm=$(( 128 + d*7*tr*8 + d*2*tr*128 + (d*tr + 512)*128 + d*tr*128 ))
  if [ $sm -le 225280 ]; then
    echo "D=$d TR=$tr smem=$sm" >> gpurun_out/r02_f_sweep.txt
    SRK_BAND_D=$d SRK_BAND_TR=$tr BAND_REPS=5 timeout 120 python scripts/band_probe.py 2>&1 | grep "gram=" >> gpurun_out/r02_f_sweep.txt
  fi
done; done
cat gpurun_out/r02_f_sweep.txt
