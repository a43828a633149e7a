#!/bin/bash
cd "$(dirname "$0")/.."
echo "base $(VD_VERBOSE=1 timeout 300 python tools/cfg4_score.py 2>&1 | tail -2)"
echo "tpp16 $(VD_VERBOSE=1 VD_TPP=16 timeout 300 python tools/cfg4_score.py 2>&1 | tail -2)"
for v in prev base; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so; echo "cfg4 GA $v"; VD_VERBOSE=1 VD_LIB=$lib timeout 600 python tools/cfg4.py 148 60 2>&1 | grep -v "^\[vd\] score" | tail -4; done
AB_ARGS="--screen-ligands 0" bash tools/ab_bench.sh prev base
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
