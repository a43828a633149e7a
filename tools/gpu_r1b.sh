#!/bin/bash
# round-1 session-2 GPU pass: GA tests, A/B, launch list, ncu captures
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"
tail -2 gpurun_out/gputests.log
bash tools/ab_bench.sh base minb3 minb4
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --screen-ligands 2000 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/r1b_score \
    python bench.py --steps 3 --warmup 3 --no-cpu --screen-ligands 0 > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/r1b_ga \
    python tools/ga_prof.py 20 > gpurun_out/ncu_ga.log 2>&1; echo "ncu ga $?"
