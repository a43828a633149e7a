#!/bin/bash
cd "$(dirname "$0")/.."
for v in base gs1 gs2; do lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  echo "$v: $(VD_LIB=$lib timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"; done
