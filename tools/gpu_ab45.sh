#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 10000"
bash tools/ab_bench.sh prev base
VD_BRICK_BUDGET_MB=200 bash tools/ab_bench.sh base | sed 's/^/bricks /'
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
