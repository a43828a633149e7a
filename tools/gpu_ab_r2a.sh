#!/bin/bash
cd "$(dirname "$0")/.."
python tools/exact_ab.py 1000 200
VD_LIB=$PWD/tmp_ab/xminb3/libvdb200.so python tools/exact_ab.py 1000 200
for cfg in "" "VD_GA_NPP=16 VD_GA_TPP=16" "VD_GA_NPP=16 VD_GA_TPP=8" "VD_GA_NPP=32 VD_GA_TPP=16"; do
  echo "== gar128 $cfg"; env $cfg VD_LIB=$PWD/tmp_ab/gar128/libvdb200.so timeout 300 python tools/cfg4.py 296 300 2>&1 | grep -E "ligands/s"
done
echo "== base"; timeout 300 python tools/cfg4.py 296 300 2>&1 | grep -E "ligands/s"
