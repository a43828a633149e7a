#!/bin/bash
cd "$(dirname "$0")/.."
for v in prev base prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "$v $(VD_LIB=$lib timeout 300 python tools/cfg4_score.py 2>&1 | tail -1)"; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
ncu --set full --import-source on --clock-control none -k regex:score_kernel -s 2 -c 1 -f -o gpurun_out/r1_cfg4_score \
    python tools/cfg4_score.py 100000 > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 $?"
