#!/bin/bash
# ncu captures for profiles/: launch list of the bench command, full set on score_kernel and ga_kernel
cd "$(dirname "$0")/.."
tag=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 2000 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/${tag}_score \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0 > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/${tag}_ga \
    python tools/ga_prof.py 20 > gpurun_out/ncu_ga.log 2>&1; echo "ncu ga $?"
