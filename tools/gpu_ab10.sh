#!/bin/bash
cd "$(dirname "$0")/.."
for v in base r128 nopipe_r168; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  echo "$v: $(VD_LIB=$lib timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"; done
echo "tpp8 r128: $(VD_GA_TPP=8 VD_LIB=tmp_ab/r128/libvdb200.so timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"
echo "tpp2 base: $(VD_GA_TPP=2 timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"
