#!/bin/bash
# reciprocal cell-index division (rsp), packed exact pose, FMA-pipe desolvation exp
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests base $?"; tail -1 gpurun_out/gputests.log
VD_LIB=tmp_ab/ppose/libvdb200.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_pp.log 2>&1; echo "tests ppose $?"; tail -1 gpurun_out/gputests_pp.log
bash tools/ab_bench.sh base
VD_NO_RSP=1 bash tools/ab_bench.sh base | sed 's/^/norsp /'
bash tools/ab_bench.sh ppose dpoly ppose_dpoly base
