#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_scoring.py -q -k alternating 2>&1 | tail -1
export AB_ARGS="--screen-ligands 0"
bash tools/ab_bench.sh base poseonly
