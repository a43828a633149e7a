#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh at10 at15 at20 at25 at30 at10
