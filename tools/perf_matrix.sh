#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# usage: tools/perf_matrix.sh lib1 [lib2 ...]  ("new" = in-tree build); every shape through every lib
for shape in "f32 1024 1080 1920 10" "f32 1 8192 8192 30" "f32 256 1080 1918" "f32 512 1080 1919" "f32 256 1081 1919" "f32crop 256 1080 1920" "u8 1024 1080 1920" "u8 512 1080 1918" "sep 1024 1080 1920" "sep 1024 1080 1918"; do
  for v in "$@"; do
    if [ "$v" = new ]; then unset HARRIS_LIB; else export HARRIS_LIB=$PWD/ab/lib$v.so; fi
    echo -n "$v "; python tools/perf_shape.py $shape
  done
done
