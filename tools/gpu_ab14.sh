#!/bin/bash
cd "$(dirname "$0")/.."
for e in "X=0" "VD_NPP=16" "VD_NPP=16 VD_L1_KB=0" "VD_NPP=16 VD_TPP=16" "VD_NPP=16 VD_TPP=16 VD_L1_KB=0" "VD_NPP=32 VD_TPP=16" "VD_NPP=16 VD_TPP=4"; do
  echo "$e: $(env $e timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"; done
