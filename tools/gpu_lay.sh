#!/bin/bash
# per-layout kernel instantiation: regression check against the last build before the plain-path work
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
export AB_ARGS="--screen-ligands 10000"
bash tools/ab_bench.sh good base good base
for v in good base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  echo "$v GA $(VD_LIB=$lib timeout 600 python tools/cfg4.py 296 60 2>&1 | grep -v scoring | grep ligands: ) | $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1 | cut -c1-60)"; done
