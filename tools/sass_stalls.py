"""Per-instruction stall reasons of an ncu report's SASS page (one kernel of the report).
    python tools/sass_stalls.py <report.ncu-rep> [min_exec] [kernel-substring]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
sub = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
blk = next(b for b in blocks if sub in b["name"])
print(blk["name"][:110])
hdr, data = blk["rows"][0], blk["rows"][1:]
ia, ie = hdr.index("Source"), hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
allc, tot = collections.Counter(), collections.Counter()
byop = collections.defaultdict(collections.Counter)
lines = []
for r in data:
    if len(r) <= max(sc) or not r[ie].isdigit():
        continue
    c = collections.Counter({hdr[i][6:]: int(r[i] or 0) for i in sc})
    allc.update(c)
    if int(r[ie]) < mn:
        continue
    tot.update(c)
    toks = r[ia].split()
    o = toks[1] if toks[0].startswith("@") else toks[0]
    byop[o.split(".")[0]].update(c)
    lines.append((sum(c.values()), r[0][-5:], r[ia][:60], c))
print("kernel stalls:", sum(allc.values()), dict(allc.most_common(8)))
print(f"exec>={mn} stalls:", sum(tot.values()), dict(tot.most_common(8)))
for o, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    print(f"{o:8s} {sum(c.values()):6d}", dict(c.most_common(4)))
print("--- top lines")
for s_, a, src, c in sorted(lines, key=lambda x: -x[0])[:20]:
    print(a, f"{src:60s}", s_, dict(c.most_common(3)))
