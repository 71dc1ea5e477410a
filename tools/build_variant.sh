#!/bin/bash
# Links paper_2510_12174_b200/libmsplat_b200_<name>.so with one source file
# recompiled under extra defines (for tools/ab_variants.sh).
# Usage: tools/build_variant.sh <name> <stem> [-DFOO=1 ...]   (after `make` in csrc/)
set -e
name=$1; stem=$2; shift 2
cd "$(dirname "$0")/../paper_2510_12174_b200/csrc"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo $ARCH -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr "$@" -c $stem.cu -o /tmp/variant_$stem.o
objs=""
for s in preprocess binning forward forward_split normals backward backward_blend optim losses trainer_ops scene_io cabi; do
  if [ $s = $stem ]; then objs="$objs /tmp/variant_$stem.o"; else objs="$objs ../../build/csrc/$s.o"; fi
done
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o ../libmsplat_b200_$name.so $objs
