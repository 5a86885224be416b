#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev: the real bench line (headline only) for the in-tree library vs ab/libold.so, alternating
for i in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export HARRIS_LIB=$PWD/ab/libold.so; else unset HARRIS_LIB; fi
    timeout 300 python bench.py --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    sleep ${PAUSE:-5}
  done
done
