#!/bin/bash
# GA A/B: concurrent vs serial buckets, register caps, pipelined gathers, TPP
cd "$(dirname "$0")/.."
bash tools/ab_bench.sh base
VD_GA_SERIAL=1 bash tools/ab_bench.sh base | sed 's/^/serial /'
bash tools/ab_bench.sh nopipe nopipe_r128 r128 nopipe_r168
VD_GA_TPP=8 bash tools/ab_bench.sh r128 nopipe_r128 | sed 's/^/tpp8 /'
VD_GA_NPP=64 bash tools/ab_bench.sh r128 nopipe_r128 | sed 's/^/npp64 /'
