"""DRAM traffic per launch of the c2 kernels from an ncu --set full report -> the JSON
bench.py reads for roofline.traffic (profiles/r2_traffic.json), keyed by kernel class and
naming the exact instantiation captured.

    python tools/ncu_traffic.py REPORT.ncu-rep OUT.json "command line of the capture"
"""
import csv
import io
import json
import subprocess
import sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
iname, ird, iwr, it = (hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"),
                       hdr.index("dram__bytes_write.sum"), hdr.index("gpu__time_duration.sum"))
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def num(v):
    return float(str(v).replace(",", ""))
cls = {"k_smooth2": "k_gs", "k_resid2": "k_proj", "k_cgp2": "k_cgp", "k_reduce_solve": "k_reduce_solve"}
acc = {}
for r in rows[2:]:
    name = r[iname]
    c = next((v for k, v in cls.items() if name.startswith(k) or ("void " + k) in name), None)
    if c is None:
        continue
    b = num(r[ird]) * scale.get(units[ird], 1e6) + num(r[iwr]) * scale.get(units[iwr], 1e6)
    t = num(r[it]) * tscale.get(units[it], 1.0)
    e = acc.setdefault(c, {"kernel": name, "n": 0, "bytes": 0.0, "us": 0.0})
    e["n"] += 1
    e["bytes"] += b
    e["us"] += t
res = {"source": f"ncu --set full --clock-control none: {cmd}; dram__bytes_read.sum + dram__bytes_write.sum "
                 f"per launch (mean over the launches captured)", "config": "c2"}
for c, e in acc.items():
    res[c] = {"kernel": e["kernel"], "dram_bytes_per_launch": e["bytes"] / e["n"],
              "ncu_time_us": e["us"] / e["n"], "launches_captured": e["n"]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
