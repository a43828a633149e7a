#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
export AB_ARGS="--screen-ligands 0"
VD_VERBOSE=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0 2>&1 | grep "\[vd\]" | sort | uniq -c | head -5
bash tools/ab_bench.sh base
VD_NO_WS=1 bash tools/ab_bench.sh base | sed 's/^/nows /'
