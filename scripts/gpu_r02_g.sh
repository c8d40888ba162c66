timeout 600 python -m pytest tests/test_gpu_band.py -q --tb=short -x 2>&1 | tail -2
for c in "0 256 16" "1 128 8"; do set -- $c
  echo "cplx=$1 m=$2 s=$3"; BAND_CPLX=$1 BAND_M=$2 BAND_S=$3 timeout 200 python scripts/band_probe.py 2>&1 | grep "gram="
  echo "ystage"; SRK_BAND_YSTAGE=1 BAND_CPLX=$1 BAND_M=$2 BAND_S=$3 timeout 200 python scripts/band_probe.py 2>&1 | grep "gram=sumvec"
done
