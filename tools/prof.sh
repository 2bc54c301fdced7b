#!/bin/bash
# One ncu --set full capture of the kernels matching a regex in a short bench run.
# usage: tools/prof.sh <kernel-regex> <tag> [count]
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${3:-1} -o gpurun_out/$2 \
  python bench.py --profile --steps 1 --warmup 1 > gpurun_out/$2.log 2>&1
tail -3 gpurun_out/$2.log
