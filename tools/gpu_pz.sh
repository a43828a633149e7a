#!/bin/bash
# A/B: z-pair loads on the plain map layout (cfg4's 126^3 grid)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in prev base prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  echo "$v $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"
  echo "$v GA $(VD_LIB=$lib timeout 600 python tools/cfg4.py 296 60 2>&1 | grep ligands: )"; done
