#!/bin/bash
cd "$(dirname "$0")/.."
VD_LIB=tmp_ab/ppose/libvdb200.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
