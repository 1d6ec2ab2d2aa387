#!/bin/bash
# C4 and C5 lag-stage timing across library builds (tools/build_variant.sh):
#   tools/ab_lag_tc.sh lib1.so lib2.so ...
cd "$(dirname "$0")/.."
for l in "$@"; do
  SA_LIB_PATH=$PWD/$l timeout 100 python tools/time_map.py 2>&1 | head -1 | sed "s|^|$l |"
  SA_LIB_PATH=$PWD/$l C5=1 timeout 100 python tools/time_map.py 2>&1 | head -1 | sed "s|^|$l |"
done
