#!/bin/bash
# like loop_md5.sh, but register numbers and addresses stripped: an unchanged
# signature means the same instruction sequence up to register renaming
L=${1:-paper_1907_11678_b200/_lib/libvelan_gpu.so}
for k in ILi0ELi1ELi15ELb1ELi2ELi5120ELb0E ILi1ELi1ELi11ELb1ELi2ELi5120ELb0E ILi1ELi1ELi15ELb1ELi2ELi5120ELb0E; do
  python tools/sass_loop.py $L $k --dump | tail -n +2 | awk '{$1=""; print}' | sed -E 's/\bU?R[0-9]+\b/R/g; s/\bU?P[0-9]\b/P/g; s/0x[0-9a-f]+/X/g' | md5sum | cut -c1-12
done | tr '\n' ' '; echo
