#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
export AB_ARGS="--screen-ligands 10000"
bash tools/ab_bench.sh prev base prev base
for v in prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "$v $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"; done
