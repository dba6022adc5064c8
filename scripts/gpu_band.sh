# banded phi exchange: tests, then interleaved A/B of kernel 3 (box) vs 5 (banded exchange) per lattice / z-chunk
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "xch" > gpurun_out/band_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/band_tests.log
for lz in ${BAND_CASES:-512,512,64:32 512,512,64:64 256,256,256:32 256,256,256:64 256,256,32:32}; do
  lat=${lz%:*}; zc=${lz#*:}
  export LB_ZCHUNK=$zc
  echo "lat=$lat zc=$zc band=${LB_XCH_BAND:-auto} $(timeout 300 python scripts/probe.py --lattice $lat --ab 3,5 --steps 20 --rounds 10 2>&1 | tail -1)"
done
unset LB_ZCHUNK
