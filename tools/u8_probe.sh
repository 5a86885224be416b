#!/bin/bash
# u8 row-group (pair / quad TMA) tile-height sweep (HARRIS_BAND_ROWS)
export HARRIS_DEV=1
for shape in "u8 512 1080 1916" "u8 512 1080 1080" "u8 256 2456 2456" "u8 512 1920 1080"; do
  for br in 0 400 538 640; do echo -n "band$br "; HARRIS_BAND_ROWS=$br python tools/perf_shape.py $shape 10; done
done
