#!/bin/bash
cd "$(dirname "$0")/.."
python tools/h2d_probe.py
export AB_ARGS="--screen-ligands 0"
for c in 32768 65536 131072 262144; do VD_CHUNK=$c bash tools/ab_bench.sh base | sed "s/^/chunk$c /"; done
