#!/bin/bash
# ncu captures of the hot kernels (each command first runs clean, then under ncu)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P=python
run() {  # name kernel-regex args...
  local name=$1 kre=$2; shift 2
  $P tools/prof_kernels.py "$@" > gpurun_out/plain_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
      -o gpurun_out/prof_$name -f $P tools/prof_kernels.py "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
for spec in "$@"; do
  IFS=: read name kre a1 a2 <<< "$spec"
  run $name $kre $a1 $a2
done
