"""Per-instruction stall reasons of the hot loop of an ncu report (SASS source page).
    python tools/sass_stalls.py <report.ncu-rep> [min_exec]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; mn = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
_sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
_all = collections.Counter()
for r in data:
    if len(r) > max(_sc):
        _all.update({hdr[i]: int(r[i] or 0) for i in _sc})
print("kernel stall totals:", sum(_all.values()), {k: v for k, v in _all.most_common() if v})
ia, ie = hdr.index("Source"), hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter(); byop = collections.defaultdict(collections.Counter)
lines = []
for r in data:
    if len(r) <= ie or not r[ie].isdigit() or int(r[ie]) < mn: continue
    c = collections.Counter({hdr[i]: int(r[i] or 0) for i in sc})
    tot.update(c)
    toks = r[ia].split(); o = toks[1] if toks[0].startswith("@") else toks[0]
    byop[o.split(".")[0]].update(c)
    lines.append((sum(c.values()), r[0][-5:], r[ia][:60], c))
print("hot-loop stall totals:", {k: v for k, v in tot.most_common() if v})
for o, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    print(f"{o:8s} {sum(c.values()):6d}", {k[6:]: v for k, v in c.most_common(4) if v})
print("--- top lines")
for s, a, src, c in sorted(lines, reverse=True)[:25]:
    print(a, f"{src:60s}", s, {k[6:]: v for k, v in c.most_common(3) if v})
