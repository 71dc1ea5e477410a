#!/bin/bash
# A/B timing of alternative builds of the kernel library on the GPU box.
# Usage: tools/ab_variants.sh <rounds> lib1.so lib2.so ...  (files under paper_2510_12174_b200/)
R=$1; shift
for i in $(seq $R); do for L in "$@"; do
  MSPLAT_LIB=$PWD/paper_2510_12174_b200/$L python tools/profile_render.py --iters 6 --timing 2>&1 | tail -1 |
    python3 -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().split('stages ')[1]); print('$L', {k: round(v[0],3) for k,v in d.items() if k in ('forward','backward','binning','preprocess','proj_bwd')})"
done; done
