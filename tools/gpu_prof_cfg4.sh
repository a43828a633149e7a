cd "$(dirname "$0")/.."
tag=r2c
C="python tools/cfg4.py 1184 3"
$C > gpurun_out/plain_c.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:ga_kernel -c 1 -f -o gpurun_out/${tag}_cfg4_ga $C > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 ga $?"
for r in cfg4_ga; do
  rep=gpurun_out/${tag}_$r.ncu-rep
  [ -f $rep ] || continue
  python tools/ncu_summary.py $rep "${tag} $r" > gpurun_out/${tag}_$r.md 2>&1
  python tools/ncu_regions.py $rep > gpurun_out/${tag}_${r}_regions.txt 2>&1
  python tools/ncu_stalls.py $rep > gpurun_out/${tag}_${r}_stalls.txt 2>&1
  ncu -i $rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $rep /tmp/ncu_reps/
done
