#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base
VD_WS=1 bash tools/ab_bench.sh base | sed 's/^/ws44 /'
VD_WS=2 bash tools/ab_bench.sh base | sed 's/^/ws26 /'
VD_WS=2 timeout 900 python -m pytest tests/test_gpu_scoring.py -x -q 2>&1 | tail -1
