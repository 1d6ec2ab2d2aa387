#!/bin/bash
# Build a variant of libsignadd_b200.so with extra -D flags into tools/variants/<name>.so:
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
root="$(cd "$(dirname "$0")/.." && pwd)"
name=$1; defs=$2
tmp=$(mktemp -d /tmp/sa_var_XXXX)
mkdir -p "$tmp/pkg"; cp -r "$root/paper_1402_0532_b200/csrc" "$tmp/pkg/csrc"
mkdir -p "$tmp/include" "$root/tools/variants"
cp "$root/include/signadd_b200.h" "$tmp/include/"
make -s -C "$tmp/pkg/csrc" -j8 NVCC="nvcc $defs" OUT="$root/tools/variants/$name.so" >/dev/null
rm -rf "$tmp"
echo "built tools/variants/$name.so ($defs)"
