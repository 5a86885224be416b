#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev sweep: L2 policy x TMA config x band rows on the probe workloads
set -u
for pol in 0 1 2; do
  HARRIS_L2_POLICY=$pol python tools/probe_perf.py --configs 0,3 --iters 20 2>&1 | sed "s/^/pol$pol /"
done
for br in 228 114 57 30; do
  HARRIS_BAND_ROWS=$br python tools/probe_perf.py --configs 0 --iters 20 2>&1 | grep 8192 | sed "s/^/rows$br /"
done
