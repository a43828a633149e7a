#!/bin/bash
# Build the library as of a git revision for A/B:  tools/ab_build_rev.sh name rev ["EXTRA"]
#   -> tmp_ab/<name>/libvdb200.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; rev=$2; flags=${3:-}
d=$ROOT/tmp_ab/$name
rm -rf "$d"; mkdir -p "$d"
git -C "$ROOT" archive "$rev" paper_2509_12232_b200/csrc include | tar -x -C "$d"
make -s -j8 -C "$d/paper_2509_12232_b200/csrc" EXTRA="$flags" OUT="$d/libvdb200.so" > "$d/build.out" 2>&1 \
  || { cat "$d/build.out"; exit 1; }
echo "built $name @ $rev"
