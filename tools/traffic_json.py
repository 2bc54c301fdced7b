"""profiles/traffic.json: dram read+write bytes per launch of each step kernel, from ncu --set full
reports (the `traffic` field of bench.py's roofline object).
    python tools/traffic_json.py <out.json> <report.ncu-rep> [...]"""
import csv
import io
import json
import subprocess
import sys

# kernel-name substring -> the bench's kernel key (KScope names)
MAP = [("TailSampleEpiT", "z2_tail_umma"), ("Gw2TEpi", "bw_gw2_umma"), ("umma2_kernel<256, 0, 1, PartialEpi", "bw_dg1_umma"),
       ("umma3p_kernel<128, 1, 1, PartialEpi, 1", "bw_gw1_umma"), ("adam_kernel", "adam"),
       ("maxcut_cut_kernel", "maxcut_energy"), ("head_v3_kernel", "head_sample"), ("dz1_kernel", "bw_dz1"),
       ("stats_weights_kernel", "stats_weights_wg1"), ("head_thresholds_kernel", "head_thresholds")]
out = {}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    hdr = rows[0]
    ki, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        name = r[ki]
        key = next((k for sub, k in MAP if sub in name), None)
        if key is None or key in out:
            continue
        b = float(r[rd].replace(",", "")) * scale.get(units[rd], 1) + float(r[wr].replace(",", "")) * scale.get(units[wr], 1)
        out[key] = b
json.dump(out, open(sys.argv[1], "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1, sort_keys=True))
