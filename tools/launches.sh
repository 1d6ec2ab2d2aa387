#!/bin/bash
# per-kernel launch times (ncu gpu__time_duration, serialised) of prof_kernels.py workloads
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in "$@"; do
  python tools/prof_kernels.py $w c64 > /dev/null 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_kernels.py $w c64 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); v=h.index('Metric Value')
for r in rows[1:]: print('$w', r[i][:70], r[v])
"
done
