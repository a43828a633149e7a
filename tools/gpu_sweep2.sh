#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
for cfg in "4 64 16" "4 64 24" "8 64 16" "8 64 32" "4 128 16" "4 128 32" "2 128 8" "2 128 16" "2 64 16" "8 32 24" "8 16 24" "4 32 12"; do
  set -- $cfg
  echo -n "TPP=$1 NPP=$2 WARPS=$3  "
  VD_TPP=$1 VD_NPP=$2 VD_WARPS=$3 bash tools/ab_bench.sh base
done
