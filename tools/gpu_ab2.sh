#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/gputests.log
bash tools/ab_bench.sh base nohint yz yznohint base
for v in base yz; do
  lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  VD_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:score_kernel -s 5 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu --screen-ligands 0 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$v /"
done
