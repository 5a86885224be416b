#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev A/B: alternate the in-tree library and ab/libharris_old.so within one box session
for i in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export HARRIS_LIB=$PWD/ab/libharris_old.so; else unset HARRIS_LIB; fi
    for c in ${CFGS:-6}; do
      HARRIS_TMA_CONFIG=$c timeout 100 python tools/variance.py ${N:-30} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); ms=d['ms']; print('$v cfg$c', 'first5', round(sum(ms[:5])/5,3), 'last10', round(sum(ms[-10:])/10,3), 'mean', round(sum(ms)/len(ms),3), 'min', min(ms), d['sm_mhz'][:3], d['reasons_or'])"
    done
  done
done
