#!/bin/bash
# r2 ncu: cfg4 GA steady state (skip the warm-up launch) and the exact-mode GA (cfg2 bucket)
cd "$(dirname "$0")/.."
tag=${1:-r2}
C="python tools/cfg4.py 296 20"
$C > gpurun_out/plain_c.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -s 1 -c 1 -f -o gpurun_out/${tag}_cfg4_ga $C > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 ga $?"
X="python tools/ga_prof.py 5 exact"
$X > gpurun_out/plain_x.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/${tag}_exact_ga $X > gpurun_out/ncu_x.log 2>&1; echo "ncu exact ga $?"
for r in cfg4_ga exact_ga; do
  rep=gpurun_out/${tag}_$r.ncu-rep
  [ -f $rep ] || continue
  python tools/ncu_summary.py $rep "${tag} $r" > gpurun_out/${tag}_$r.md 2>&1
  python tools/ncu_regions.py $rep > gpurun_out/${tag}_${r}_regions.txt 2>&1
  python tools/ncu_stalls.py $rep > gpurun_out/${tag}_${r}_stalls.txt 2>&1
  ncu -i $rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $rep /tmp/ncu_reps/
done
