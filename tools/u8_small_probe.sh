#!/bin/bash
# single-frame tile-height sweep (graph replay) for u8 and f32 frames
export HARRIS_DEV=1
for hw in "1536 2560" "2832 4256"; do
  for br in 0 64 128 192 256 384; do HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py $hw; done
  for br in 0 48 64 96 128 192; do HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py $hw f32; done
  for br in 0 64 128; do HARRIS_TMA_CONFIG=6 HARRIS_BAND_ROWS=$br python tools/u8_small_probe.py $hw f32; done
done
