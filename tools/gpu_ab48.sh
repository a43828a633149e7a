#!/bin/bash
cd "$(dirname "$0")/.."
echo "score: $(timeout 300 python tools/score_bucket.py 2>&1 | tail -1)"
echo "ga:    $(timeout 300 python tools/ga_bucket.py 2>&1 | tail -1)"
