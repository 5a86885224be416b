#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev A/B of sustained behaviour: N back-to-back launches (tools/variance.py), new vs ab/libharris_old.so
for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export HARRIS_LIB=$PWD/ab/libharris_old.so; else unset HARRIS_LIB; fi
    for c in ${CFGS:-6}; do
      HARRIS_TMA_CONFIG=$c timeout 200 python tools/variance.py ${N:-80} > gpurun_out/var_tmp.txt 2>&1
      python -c "
import json
d=json.loads(open('gpurun_out/var_tmp.txt').read().strip().splitlines()[-1]); ms=d['ms']
print('$v cfg$c', 'bench-window(3:23)', round(sum(ms[3:23])/20,3), 'first5', round(sum(ms[:5])/5,3), 'last20', round(sum(ms[-20:])/20,3), 'min', min(ms), 'sm', d['sm_mhz'][-3:], d.get('reasons_or'))"
    done
  done
done
