#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/gputests.log
for v in cta0 wl0; do VD_LIB=tmp_ab/$v/libvdb200.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$v.log 2>&1; echo "tests $v $?"; done
bash tools/ab_bench.sh base prev wl0 cta0 base prev wl0 cta0
