#!/bin/bash
cd "$(dirname "$0")/.."
ncu --set full --import-source on --clock-control none -k regex:score_ws_kernel -s 5 -c 1 -f -o gpurun_out/ws_score \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0 > gpurun_out/ncu_ws.log 2>&1; echo "ncu ws $?"
