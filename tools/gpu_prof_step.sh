#!/bin/bash
# ncu source-level capture of ga_step_kernel (cfg2 33-48-atom ligands)
cd "$(dirname "$0")/.."
G="python tools/ga_prof.py 6"
$G > gpurun_out/plain_g.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_step_kernel -s 4 -c 1 -f -o gpurun_out/step $G > gpurun_out/ncu_step.log 2>&1; echo "ncu $?"
ncu -i gpurun_out/step.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/step_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/step.ncu-rep "ga_step 64 regs" > gpurun_out/step.md 2>&1
rm -f gpurun_out/step.ncu-rep
