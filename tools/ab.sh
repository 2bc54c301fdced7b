#!/bin/bash
# A/B of an env toggle on the 1-GPU bench: tools/ab.sh VAR valA valB [rounds]
b() { python bench.py --no-cpu-baseline --steps 40 --warmup 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for r in $(seq ${4:-3}); do
  echo "$1=$2 $(env $1=$2 bash -c "$(declare -f b); b")  $1=$3 $(env $1=$3 bash -c "$(declare -f b); b")"
done
