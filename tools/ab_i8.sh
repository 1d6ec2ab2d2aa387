#!/bin/bash
# A/B of sa_ndft_i8 variants (tools/build_variant.sh): C2 c128 tc timing + parity of each
cd "$(dirname "$0")/.."
for l in "$@"; do
  SA_LIB_PATH=$PWD/$l timeout 200 python tools/time_ndft_i8.py 2>&1 | grep " tc" | tail -1 | sed "s|^|$l |"
  SA_LIB_PATH=$PWD/$l timeout 300 python -m pytest tests/test_gpu_ndft_i8.py -q -m gpu -p no:cacheprovider -k "sizes or dynamic" 2>&1 | tail -1 | sed "s|^|$l |"
done
