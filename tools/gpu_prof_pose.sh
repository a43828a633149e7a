#!/bin/bash
# ncu source-level capture of the pose stage alone (timing build: energy stage compiled out)
cd "$(dirname "$0")/.."
VD_LIB=tmp_ab/poseonly/libvdb200.so ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 5 -c 1 -f -o gpurun_out/pose_only \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --screen-ligands 0 > gpurun_out/ncu_pose.log 2>&1; echo "ncu pose $?"
