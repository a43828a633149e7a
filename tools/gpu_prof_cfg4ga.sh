#!/bin/bash
# ncu capture of the cfg4 GA kernel (128-atom ligands, pop 512, 20 generations)
cd "$(dirname "$0")/.."
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/cfg4_ga \
    python tools/cfg4.py 296 20 > gpurun_out/ncu_cfg4ga.log 2>&1; echo "ncu cfg4 ga $?"
