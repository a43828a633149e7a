#!/bin/bash
# Build variant libraries for compile-time A/B on the GPU box:
#   tools/ab_build.sh name "EXTRA flags" [name "flags" ...]  ->  tmp_ab/<name>/libvdb200.so
# then run with VD_LIB=tmp_ab/<name>/libvdb200.so (paper_2509_12232_b200/_abi.py).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=$ROOT/tmp_ab/$name
  rm -rf "$d"; mkdir -p "$d/pkg"
  ln -s "$ROOT/include" "$d/include"
  cp -r "$ROOT/paper_2509_12232_b200/csrc" "$d/pkg/csrc"
  rm -rf "$d/pkg/csrc/build"
  make -s -j8 -C "$d/pkg/csrc" EXTRA="$flags" OUT="$d/libvdb200.so" "$d/libvdb200.so" > "$d/build.out" 2>&1 \
    || { cat "$d/build.out"; exit 1; }
  echo "built $name ($flags)"
done
