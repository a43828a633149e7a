#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
python tools/diag_e2e.py 2>&1 | tail -5
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh prev base prev base
