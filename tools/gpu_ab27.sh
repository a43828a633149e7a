#!/bin/bash
cd "$(dirname "$0")/.."
echo "npp64 base: $(VD_GA_NPP=64 VD_VERBOSE=1 timeout 300 python tools/ga_bucket.py 2>&1 | grep -v '^\[vd\] score' | tail -5)"
echo "npp64 gs1: $(VD_GA_NPP=64 VD_LIB=tmp_ab/gs1/libvdb200.so timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"
