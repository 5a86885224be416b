#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev: f32 default config device time for several library variants (HARRIS_LIB), alternating
for i in 1 2; do
  for v in ${VARIANTS:-new old}; do
    if [ $v = new ]; then unset HARRIS_LIB; else export HARRIS_LIB=$PWD/ab/lib$v.so; fi
    echo "== $v"
    timeout 200 python tools/probe_perf.py --configs ${F32CFG:-6} --iters 30 2>&1 | grep -v " 1x1536x2560"
  done
done
