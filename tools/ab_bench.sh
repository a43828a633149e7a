#!/bin/bash
# A/B of variant libraries (tools/ab_build.sh) on the bench: kernel ms, screening ligands/s.
#   tools/ab_bench.sh base minb3 ...   ("base" = the in-tree library)
for v in "$@"; do
  lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  VD_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-extra ${AB_ARGS:-} > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.log").read().strip().splitlines()[-1])
    s = d.get("screening", {})
    print(f"{v:12s} {d['ms_per_step']:.4f} ms  {d['value']/1e6:.1f} M poses/s  e2e {d['e2e']['value']/1e6:.1f}  "
          f"screen {s.get('value', 0):.0f} lig/s  parity {d['parity_sample_ok']}  sm {d['clocks']['sm_mhz']}")
except Exception as e:
    print(v, "FAILED", e)
PY
done
