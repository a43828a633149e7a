#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/ab_bench.sh base split1 split2 split3 base
