#!/usr/bin/env python
"""The north-star N sweep (BASELINE.json configs): one bench.py run per configuration on 1 GPU,
recording samples/s, steps/s, e2e, the roofline line, the final cut and the reference CPU
baseline measured beside it on the same host (full steps where they fit in the budget, else
the per-bit extrapolation).

    python scripts/n_sweep.py [--out profiles/nsweep.json] [--steps 20]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [  # (N, graph, note) -- BASELINE.json configs[0..4] and the G(n,3/4) stress variant
    (20, "regular3", "configs[0]: random 3-regular N=20"),
    (100, "regular3", "configs[1]: random 3-regular N=100"),
    (1000, "maxcut", "configs[2]: N=1000 with the reference's random_maxcut_graph G(n,3/4)"),
    (5000, "regular3", "configs[3]: random regular N=5000"),
    (10000, "regular3", "configs[4]: random 3-regular N=10000 (headline)"),
    (10000, "maxcut", "stress: the reference generator's G(10^4, 3/4), |E| ~ 3.75e7"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args()
    rows = []
    for n, graph, note in CONFIGS:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--n", str(n), "--graph", graph, "--steps",
               str(a.steps), "--warmup", "5", "--no-sr", "--cpu-seconds", str(a.cpu_seconds)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            rows.append(dict(n=n, graph=graph, note=note, error=r.stderr[-2000:]))
            print(json.dumps(rows[-1]), flush=True)
            continue
        cpu = d.get("cpu_baseline") or {}
        row = dict(n=n, graph=graph, note=note, workload=d["config"]["workload"], samples_per_s=d["value"],
                   steps_per_s=d.get("steps_per_s"), ms_per_step=d["ms_per_step"], e2e=d.get("e2e", {}).get("value"),
                   roofline=d.get("roofline"), head_latency=d.get("head_latency"), final_cut=d.get("final_cut"),
                   clocks=d.get("clocks"), cpu_baseline=cpu,
                   speedup_vs_cpu=(d["value"] / cpu["value"]) if cpu.get("value") else None)
        rows.append(row)
        print(json.dumps({k: row[k] for k in ("n", "graph", "samples_per_s", "ms_per_step", "e2e", "speedup_vs_cpu")}),
              flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"device": "B200 (1 GPU)", "configs": rows}, f, indent=1)


if __name__ == "__main__":
    main()
