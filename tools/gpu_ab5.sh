#!/bin/bash
cd "$(dirname "$0")/.."
VD_LIB=tmp_ab/nopipe/libvdb200.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -1 gpurun_out/gputests.log
bash tools/ab_bench.sh base nopipe
VD_NPP=64 bash tools/ab_bench.sh nopipe
VD_NPP=16 bash tools/ab_bench.sh nopipe
