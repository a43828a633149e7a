#!/bin/bash
cd "$(dirname "$0")/.."
run() { echo "$1: $(env $2 VD_LIB=$3 timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"; }
run base "X=0" ""
run "gr128 tpp8" "VD_GA_TPP=8" tmp_ab/gr128/libvdb200.so
run "gr128np tpp8" "VD_GA_TPP=8" tmp_ab/gr128np/libvdb200.so
run "gs1" "X=0" tmp_ab/gs1/libvdb200.so
run "gr128 tpp4" "X=0" tmp_ab/gr128/libvdb200.so
