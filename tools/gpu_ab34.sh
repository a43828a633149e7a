#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh prev base
VD_NPP=32 VD_TPP=8 bash tools/ab_bench.sh lb3 base | sed 's/^/32x8 /'
VD_NPP=32 VD_TPP=4 bash tools/ab_bench.sh base | sed 's/^/32x4 /'
bash tools/ab_bench.sh prev base
