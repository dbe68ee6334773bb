#!/bin/bash
# usage: tools/ncu_capture.sh <kernel-regex> <out-name> [skip]  — one full ncu capture of a bench launch
K=$1; O=$2; S=${3:-7}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/$O \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/$O.log 2>&1
echo "ncu $O rc=$?"
