#!/bin/bash
# isolated (plain, no PDL overlap) single frames: tile-height sweep
export HARRIS_DEV=1
for br in 0 48 64 96 128; do
  HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py 1536 2560 f32 plain | sed "s/^/band$br /"
  HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py 1536 2560 u8 plain | sed "s/^/band$br /"
  HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py 2832 4256 f32 plain | sed "s/^/band$br /"
done
