#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh r26 r30 r36 r45 r26
