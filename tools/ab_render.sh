#!/bin/bash
# Render A/B of library variants: tools/ab_render.sh name1 name2 ...
for v in "$@"; do
  echo "== $v"
  TFG_LIB=paper_2507_01631_b200/_variants/$v/libtilefield_gpu.so timeout 200 python tools/time_render.py 2>&1 | tail -1
done
