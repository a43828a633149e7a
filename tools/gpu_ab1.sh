#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/gputests.log
bash tools/ab_bench.sh base old nofused nolerp minb3 base
