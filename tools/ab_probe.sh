#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev A/B: in-tree library vs ab/libharris_old.so, alternating, f32 and u8 default configs
for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export HARRIS_LIB=$PWD/ab/libharris_old.so; else unset HARRIS_LIB; fi
    echo "== $v"
    timeout 200 python tools/probe_perf.py --configs ${F32CFG:-6} --iters 30 2>&1 | grep -v " 1x1536x2560"
    timeout 200 python tools/probe_perf.py --u8 --configs ${U8CFG:-5} --iters 20 2>&1 | grep -v " 1x1536x2560"
  done
done
