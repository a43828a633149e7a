#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
VD_WS=3 bash tools/ab_bench.sh base | sed 's/^/ws17 /'
bash tools/ab_bench.sh base
