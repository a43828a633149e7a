#!/bin/bash
# r2 ncu captures for profiles/: bench launch list; full set on score_kernel (cfg1), ga_kernel
# (cfg2 33-48-atom bucket) and ga_kernel (cfg4).  Each command runs once plainly first.
cd "$(dirname "$0")/.."
tag=${1:-r2}
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 2000"
[ -n "$SKIP_RUN" ] || $B > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
S="python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0"
$S > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/${tag}_score $S > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
G="python tools/ga_prof.py 20"
$G > gpurun_out/plain_g.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/${tag}_ga $G > gpurun_out/ncu_ga.log 2>&1; echo "ncu ga $?"
C="python tools/cfg4.py 296 20"
$C > gpurun_out/plain_c.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/${tag}_cfg4_ga $C > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 ga $?"
# summarise on the box (the full-set reports exceed gpurun's 64 MiB copy-back limit)
for r in score ga cfg4_ga; do
  rep=gpurun_out/${tag}_$r.ncu-rep
  [ -f $rep ] || continue
  python tools/ncu_summary.py $rep "${tag} $r" $([ $r = score ] && echo gpurun_out/${tag}_launches.csv) > gpurun_out/${tag}_$r.md 2>&1
  python tools/ncu_regions.py $rep > gpurun_out/${tag}_${r}_regions.txt 2>&1
  python tools/ncu_stalls.py $rep > gpurun_out/${tag}_${r}_stalls.txt 2>&1
  ncu -i $rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $rep /tmp/ncu_reps/
done
du -sh gpurun_out
