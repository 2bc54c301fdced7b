#!/bin/bash
# ncu launch list (per-kernel gpu__time_duration, cold-cache serialised) of a short bench run.
# usage: tools/launches.sh <tag>
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$1_launches.csv \
  python bench.py --profile --steps 2 --warmup 1 > gpurun_out/$1_ncu_launch.log 2>&1
python tools/ncu_summary.py launches gpurun_out/$1_launches.csv gpurun_out/$1_launches.txt > /dev/null; cat gpurun_out/$1_launches.txt
