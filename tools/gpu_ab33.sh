#!/bin/bash
cd "$(dirname "$0")/.."
for v in base st512 st1024; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  echo "$v $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"
  echo "$v tpp16 $(VD_TPP=16 VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"
  echo "$v GA $(VD_LIB=$lib timeout 600 python tools/cfg4.py 148 60 2>&1 | grep ligands: )"
done
