#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -1 gpurun_out/gputests.log
VD_LIB=tmp_ab/nopipe/libvdb200.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests2.log 2>&1; echo "tests nopipe $?"; tail -1 gpurun_out/gputests2.log
bash tools/ab_bench.sh base nopipe prev base nopipe prev
