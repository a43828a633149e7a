#!/bin/bash
# ncu --set full of the bench's score_kernel (one launch after warm-up)
cd "$(dirname "$0")/.."
tag=${1:-r1d}
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/${tag}_score \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0 > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
