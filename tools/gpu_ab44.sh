#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base
VD_BRICK_BUDGET_MB=200 bash tools/ab_bench.sh base | sed 's/^/bricks /'
