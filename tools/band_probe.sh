#!/bin/bash
# stencil tile-height sweep (HARRIS_BAND_ROWS) over several plane shapes
export HARRIS_DEV=1
for shape in "sep 1024 1080 1920" "sep 16 8192 8192" "sep 256 1536 2560" "sep 4096 512 512" "sepcrop 1024 1080 1922"; do
  for br in 0 112 124 136 148 160; do echo -n "band$br "; HARRIS_BAND_ROWS=$br python tools/perf_shape.py $shape 10; done
done
