#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev: unaligned-input (K2) timing for several library variants
for i in 1 2; do
  for v in ${VARIANTS}; do
    export HARRIS_LIB=$PWD/ab/lib$v.so
    echo "== $v"; timeout 200 python tools/probe_generic.py 2>&1 | grep "auto" | grep -v "8192x8192\|1920 "
  done
done
