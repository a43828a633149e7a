#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -1 gpurun_out/gputests.log
bash tools/ab_bench.sh base prev base
for v in base prev; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "cfg4 $v"; VD_LIB=$lib timeout 600 python tools/cfg4.py 64 50 2>&1 | tail -2; done
