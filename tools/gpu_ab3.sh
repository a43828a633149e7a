#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/gputests.log
bash tools/ab_bench.sh base prev base prev
