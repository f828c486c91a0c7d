#!/bin/bash
# Build an A/B variant of the library with extra nvcc defines:
#   tools/build_variant.sh <name> -DFOO=1 ...  ->  _lib/variants/libflashfps_b200_<name>.so
# (load it with FFPS_LIB_VARIANT=<name>)
set -e
name=$1; shift
src=$(cd "$(dirname "$0")/../paper_2604_17720_b200/csrc" && pwd)
out=$src/../_lib/variants
mkdir -p $out/obj_$name
objs=""
for f in $src/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o $out/obj_$name/$b.o &
  objs="$objs $out/obj_$name/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libflashfps_b200_$name.so $objs
echo built $out/libflashfps_b200_$name.so
