#!/bin/bash
cd "$(dirname "$0")/.."
VD_LIB=tmp_ab/srcp/libvdb200.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
export AB_ARGS="--screen-ligands 10000"
bash tools/ab_bench.sh base srcp base srcp
