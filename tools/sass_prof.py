"""Summarise an ncu report's SASS page: instruction mix, top stall lines, stall reasons.
    python tools/sass_prof.py <report.ncu-rep> [kernel-index]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# split by kernel blocks (each begins with a "Kernel Name" row)
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blk = blocks[k]
hdr, data = blk["rows"][0], blk["rows"][1:]
ia, ie, isamp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
print(blk["name"][:120])
op, st, tot, tots = collections.Counter(), collections.Counter(), 0, 0
for r in data:
    try:
        n = int(r[ie]); sm = int(r[isamp] or 0)
    except (ValueError, IndexError):
        continue
    toks = r[ia].split()
    if not toks:
        continue
    o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    o = o.split(".")[0]
    op[o] += n; st[o] += sm; tot += n; tots += sm
print("instructions", tot, "stall samples", tots)
for o, n in op.most_common(25):
    print(f"{o:10s} {n:12d} {n / tot:6.3f}  stall {st[o] / max(tots, 1):6.3f}")
print("--- top stall lines")
top = sorted(data, key=lambda r: -int(r[isamp]) if len(r) > isamp and r[isamp].isdigit() else 0)[:30]
for r in top:
    print(r[0][-6:], f"{r[ia][:70]:70s}", r[isamp], r[ie])
