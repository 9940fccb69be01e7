#!/bin/bash
# Build libspmmm variants with extra nvcc defines into variants/<name>/libspmmm.so
#   tools/build_variants.sh name1:"-DX=1 -DY=1" name2:"..."
set -e
cd "$(dirname "$0")/../paper_1303_1651_b200/csrc"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  out=../../variants/$name
  mkdir -p $out
  make -s -j8 OBJDIR=$out/obj OUT=$out/libspmmm.so NVFLAGS="-O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC,-O2 -gencode arch=compute_100a,code=sm_100a $defs" >/dev/null
  echo "built $name ($defs)"
done
