#!/bin/bash
# A/B of env overrides on the cfg1 bench kernel only (no screening / extra legs)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  [ "$cfg" = base ] && cfg=""
  env $cfg timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-extra --screen-ligands 0 > gpurun_out/ab.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1].ljust(40), round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,1), 'M/s', d['parity_sample_ok'], d['clocks']['sm_mhz'])" "${cfg:-base}" || tail -5 gpurun_out/ab.log
done
