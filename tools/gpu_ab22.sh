#!/bin/bash
cd "$(dirname "$0")/.."
VD_VERBOSE=1 timeout 300 python tools/score_bucket.py 2>&1 | tail -6
