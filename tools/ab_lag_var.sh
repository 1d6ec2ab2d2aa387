#!/bin/bash
# lag-stage variants (tools/variants/NAME.so) vs the in-tree library: C4 and C5 map timing
cd "$(dirname "$0")/.."
for v in base "$@"; do
  for c5 in 0 1; do
    if [ $v = base ]; then L=""; else L=$PWD/tools/variants/$v.so; fi
    SA_LIB_PATH=$L C5=$c5 timeout 300 python tools/time_map.py 2>&1 | sed "s/^/$v /" | grep -v complex128
  done
done
