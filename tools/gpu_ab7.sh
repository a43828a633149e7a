#!/bin/bash
cd "$(dirname "$0")/.."
export AB_ARGS="--screen-ligands 0"
for cv in 50 66 75 100; do echo "carveout $cv"; VD_CARVEOUT=$cv bash tools/ab_bench.sh base nopipe; done
