#!/bin/bash
# Build an A/B variant of the library into ab/lib<name>.so with extra nvcc defines:
#   tools/build_variant.sh <name> -DFOO=1 ...   (then HARRIS_LIB=$PWD/ab/lib<name>.so)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2212_12035_b200/csrc"
out=../../ab/build_$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -ccbin /usr/bin/g++ $*"
objs=""
for f in harris_abi harris_tma harris_u8 harris_generic harris_synth harris_groupings harris_groupings_tma stencil_sep harris_peer harris_ldg; do
  $NV -c $f.cu -o $out/$f.o &
  objs="$objs $out/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../ab/lib$name.so $objs
echo built ab/lib$name.so
