#!/bin/bash
# full bench line + launch list + ncu --set full of score_kernel and ga_kernel
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"; cat gpurun_out/bench.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
bash tools/gpu_prof.sh ${1:-r1f}
