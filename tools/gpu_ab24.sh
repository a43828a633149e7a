#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base ps0 base ps0
