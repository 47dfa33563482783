#!/bin/bash
# Window-move A/B of library variants: tools/ab_window.sh name1 name2 ...
for v in "$@"; do
  echo "== $v"
  TFG_LIB=paper_2507_01631_b200/_variants/$v/libtilefield_gpu.so timeout 150 python tools/time_accept.py 2>&1 | tail -2
done
