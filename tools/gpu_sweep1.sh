#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
for cfg in "4 32 12" "4 32 8" "4 32 16" "8 16 12" "8 16 8" "8 16 16" "4 16 12" "4 16 8" "8 32 8" "8 32 16" "2 32 12" "2 64 12" "4 64 16" "4 64 8"; do
  set -- $cfg
  echo -n "TPP=$1 NPP=$2 WARPS=$3  "
  VD_TPP=$1 VD_NPP=$2 VD_WARPS=$3 bash tools/ab_bench.sh base
done
