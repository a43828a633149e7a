#!/bin/bash
# A/B of launch-shape overrides on the bench kernel (one GPU box, back to back)
for cfg in "$@"; do
  env $cfg timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1].ljust(40), round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M/s', d['parity_sample_ok'], d['clocks']['sm_mhz'])" "$cfg"
done
