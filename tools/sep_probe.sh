#!/bin/bash
# stencil pipeline-shape sweep (HARRIS_SEP_CONFIG) on contiguous 1918-wide outputs and the
# aligned crop case; band height and the per-tile CTA barrier on the default config
export HARRIS_DEV=1
for cfg in 0 4 5 6 7 8 1; do
  for shape in "sep 1024 1080 1920" "sepcrop 1024 1080 1922"; do
    echo -n "cfg$cfg "; HARRIS_SEP_CONFIG=$cfg python tools/perf_shape.py $shape 10
  done
done
for br in 136 538 1078; do echo -n "band$br "; HARRIS_SEP_CONFIG=0 HARRIS_BAND_ROWS=$br python tools/perf_shape.py sep 1024 1080 1920 10; done
echo -n "nosync "; HARRIS_SEP_CONFIG=0 HARRIS_SYNC_WAVES=0 python tools/perf_shape.py sep 1024 1080 1920 10
