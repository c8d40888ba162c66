# banded vector kernel (A^H p of the economic variants): parity, bench path, default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_benchpath.py -q --tb=short > gpurun_out/r02y_band.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_band.log
timeout 900 python bench.py --no-cpu > gpurun_out/r02y_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_bench.log
SRK_NO_BAND_VEC=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r02y_bench_novec.log 2>&1
tail -n 5 gpurun_out/r02y_band.log
for f in r02y_bench r02y_bench_novec; do grep "^{" gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), [(k['kernel'], round(k['avg_launch_ms'],3), k['frac'] and round(k['frac'],3)) for k in d['iteration']['kernels'][:7]])"; done
