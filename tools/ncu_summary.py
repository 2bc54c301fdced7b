"""Summarise ncu reports / launch lists into profiles/*.txt (committed evidence).

    python tools/ncu_summary.py launches <launches.csv> [<out>]
    python tools/ncu_summary.py report <file.ncu-rep> [<out>]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, rows = r, rows[i + 1:]
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("<")[0][-60:]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = io.StringIO()
    out.write(f"# ncu launch list: {path}\n# gpu__time_duration.sum (ns), cold-cache serialised; compare shares\n")
    out.write(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.write(f"{k:60s} {cnt[k]:8d} {tot[k] / 1e3:10.2f} {tot[k] / cnt[k] / 1e3:9.2f} {tot[k] / s:7.3f}\n")
    return out.getvalue()


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = io.StringIO()
    out.write(f"# ncu --set full: {path}\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.write(f"\n## {name[:120]}\n")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.write(f"{k:70s} {r[i]:>16s} {units[i]}\n")
    return out.getvalue()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    text = launches(path) if mode == "launches" else report(path)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(text)
    print(text)
