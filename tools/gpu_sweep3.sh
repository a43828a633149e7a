#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
for cfg in "4 48 18" "4 48 12" "4 64 16"; do
  set -- $cfg
  echo -n "TPP=$1 NPP=$2 WARPS=$3  "
  VD_TPP=$1 VD_NPP=$2 VD_WARPS=$3 bash tools/ab_bench.sh base
done
for n in 32 64 16; do echo -n "GA NPP=$n "; VD_GA_NPP=$n AB_ARGS="" bash tools/ab_bench.sh base; done
