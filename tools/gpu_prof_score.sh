#!/bin/bash
# one ncu --set full capture of the cfg1 score kernel (+ raw CSV, regions, stalls)
cd "$(dirname "$0")/.."
tag=${1:-r2s}
S="python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0"
$S > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/${tag}_score $S > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
rep=gpurun_out/${tag}_score.ncu-rep
python tools/ncu_summary.py $rep "${tag} score" > gpurun_out/${tag}_score.md 2>&1
python tools/ncu_regions.py $rep > gpurun_out/${tag}_score_regions.txt 2>&1
python tools/ncu_stalls.py $rep > gpurun_out/${tag}_score_stalls.txt 2>&1
ncu -i $rep --page raw --csv > gpurun_out/${tag}_score_raw.csv 2>/dev/null
ncu -i $rep --page source --csv > gpurun_out/${tag}_score_source.csv 2>/dev/null
mkdir -p /tmp/ncu_reps && mv $rep /tmp/ncu_reps/
du -sh gpurun_out
