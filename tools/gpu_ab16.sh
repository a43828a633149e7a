#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
for v in prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "cfg4 GA $v"; VD_LIB=$lib timeout 600 python tools/cfg4.py 148 60 2>&1 | tail -2; done
