#!/bin/bash
# frame-stream planning: HARRIS_STREAM_SHARE (frames planned for 1/share of the GPU)
export HARRIS_DEV=1
for sh in 1 2 4 8 16; do
  for hw in "1536 2560" "2832 4256"; do
    HARRIS_STREAM_SHARE=$sh python tools/u8_small_probe.py $hw f32 independent,graph,frames,plain
    HARRIS_STREAM_SHARE=$sh python tools/u8_small_probe.py $hw u8 independent,graph,frames
  done
done
