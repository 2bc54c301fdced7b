#!/bin/bash
# Sweep one env knob over values on the 1-GPU bench (ms per step, 2 runs each): tools/sweep.sh VAR v1 v2 ...
var=$1; shift
b() { python bench.py --no-cpu-baseline --steps 40 --warmup 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],5))"; }
for v in "$@"; do
  echo "$var=$v $(env $var=$v bash -c "$(declare -f b); b") $(env $var=$v bash -c "$(declare -f b); b")"
done
