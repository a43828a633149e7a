#!/bin/bash
for c in "$@"; do
  VD_CHUNK=$c timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu --screen-ligands 0 > gpurun_out/e2e.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/e2e.log').read().strip().splitlines()[-1]);print('chunk',sys.argv[1], round(d['e2e']['value']/1e6,1),'M/s e2e', round(d['value']/1e6,1),'M/s kernel')" "$c"
done
