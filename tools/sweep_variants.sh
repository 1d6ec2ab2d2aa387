#!/bin/bash
# time tools/time_ndft.py against each tools/variants/lib_*.so
cd "$(dirname "$0")/.."
for f in tools/variants/lib_*.so; do
  echo "== $f"; SA_LIB_PATH=$PWD/$f timeout 120 python tools/time_ndft.py 2>&1 | head -1
done
