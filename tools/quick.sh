#!/bin/bash
# Iteration helper for the GPU box: GPU tests, then a short bench with a one-line summary.
# usage: tools/quick.sh [pytest-args...]
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("MS", round(d["ms_per_step"], 4), round(d["value"]), "e2e", round(d["e2e"]["value"]), "clk", d["clocks"])
print({k: v["avg_ms"] for k, v in d["kernels"].items()})
PY
