#!/bin/bash
cd "$(dirname "$0")/.."
AB_ARGS="--screen-ligands 0" bash tools/ab_bench.sh prev base rsp0 ppose prev base rsp0 ppose
for v in prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "$v $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"; done
