#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base
VD_TPP=8 bash tools/ab_bench.sh base ni3 ni5 ni6 | sed 's/^/tpp8 /'
VD_NPP=32 bash tools/ab_bench.sh base ni5 | sed 's/^/npp32 /'
bash tools/ab_bench.sh ni5 ni6 base
