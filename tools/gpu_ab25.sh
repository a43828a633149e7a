#!/bin/bash
cd "$(dirname "$0")/.."
echo "bricks $(timeout 300 python tools/score_bucket.py 2>&1 | tail -1)"
echo "zy     $(VD_BRICK_BUDGET_MB=0 timeout 300 python tools/score_bucket.py 2>&1 | tail -1)"
export AB_ARGS="--screen-ligands 10000"
bash tools/ab_bench.sh base
VD_BRICK_BUDGET_MB=0 bash tools/ab_bench.sh base | sed 's/^/zy /'
