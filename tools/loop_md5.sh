#!/bin/bash
# md5 of the hot trace loops (CMP-L, CRS-S, CRS-L instantiations) of the built
# library: an edit outside the loop that leaves these unchanged cannot have
# moved ptxas's schedule of the loop
L=${1:-paper_1907_11678_b200/_lib/libvelan_gpu.so}
for k in ILi0ELi1ELi15ELb1ELi2ELi5120 ILi1ELi1ELi11ELb1ELi2ELi5120 ILi1ELi1ELi15ELb1ELi2ELi5120; do
  python tools/sass_loop.py $L $k --dump | md5sum | cut -c1-12
done | tr '\n' ' '; echo
