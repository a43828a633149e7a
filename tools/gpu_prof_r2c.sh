#!/bin/bash
# round-2 final ncu captures for profiles/: bench launch list; full set on score_kernel (cfg1),
# pop_score_kernel + ga_step_kernel (cfg2 33-48-atom ligands, generation-synchronous GA) and the
# persistent ga_kernel (cfg4, 16 subs, cp.async pair tiles).  Each command runs plainly first.
cd "$(dirname "$0")/.."
tag=${1:-r2c}
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 2000"
$B > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
S="python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0"
$S > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/${tag}_score $S > gpurun_out/ncu_score.log 2>&1; echo "ncu score $?"
G="python tools/ga_prof.py 6"
$G > gpurun_out/plain_g.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:pop_score_kernel -s 4 -c 1 -f -o gpurun_out/${tag}_pop_score $G > gpurun_out/ncu_pop.log 2>&1; echo "ncu pop_score $?"
ncu --set full --import-source on --clock-control none -k regex:ga_step_kernel -s 4 -c 1 -f -o gpurun_out/${tag}_ga_step $G > gpurun_out/ncu_step.log 2>&1; echo "ncu ga_step $?"
C="python tools/cfg4.py 296 20"
$C > gpurun_out/plain_c.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -s 1 -c 1 -f -o gpurun_out/${tag}_cfg4_ga $C > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 ga $?"
for r in score pop_score ga_step cfg4_ga; do
  rep=gpurun_out/${tag}_$r.ncu-rep
  [ -f $rep ] || continue
  python tools/ncu_summary.py $rep "${tag} $r" $([ $r = score ] && echo gpurun_out/${tag}_launches.csv) > gpurun_out/${tag}_$r.md 2>&1
  python tools/ncu_regions.py $rep > gpurun_out/${tag}_${r}_regions.txt 2>&1
  python tools/ncu_stalls.py $rep > gpurun_out/${tag}_${r}_stalls.txt 2>&1
  ncu -i $rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $rep /tmp/ncu_reps/
done
du -sh gpurun_out
