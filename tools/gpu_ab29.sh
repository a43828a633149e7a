#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base wsnoseq
VD_NO_WS=1 bash tools/ab_bench.sh base | sed 's/^/nows /'
bash tools/ab_bench.sh base
