#!/bin/bash
# cfg4 A/B of GA / score launch shapes (env overrides); usage: bash tools/gpu_cfg4_ab.sh N GENS
cd "$(dirname "$0")/.."
N=${1:-296}; G=${2:-300}
for cfg in "" "VD_GA_TPP=16" "VD_GA_TPP=16 VD_GA_NPP=32" "VD_GA_TPP=16 VD_TPP=16" "VD_TPP=16 VD_NPP=16"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/cfg4.py $N $G 2>&1 | grep -E "ligands/s|scoring"
done
