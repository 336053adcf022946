"""Per-launch DRAM traffic of a captured kernel (ncu --set full report) for bench.py's
`roofline.traffic`: writes/updates profiles/traffic.json[workload].

    python tools/traffic_summary.py <report.ncu-rep> <workload> <algorithmic_bytes> <note>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, workload, alg, note = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
d = dict(zip(h, rows[2]))


def num(k):
    return float(d[k].replace(",", ""))


BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
SECONDS = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
           "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def scaled(k, table):
    return num(k) * table[rows[1][h.index(k)]]


rd, wr = scaled("dram__bytes_read.sum", BYTES), scaled("dram__bytes_write.sum", BYTES)
scale = 1.0
dur, dscale = scaled("gpu__time_duration.sum", SECONDS), 1.0
entry = {"kernel": d["Kernel Name"][:200], "grid": d.get("Grid Size"), "block": d.get("Block Size"),
         "dram_bytes_per_launch": (rd + wr) * scale, "dram_read_bytes": rd * scale,
         "dram_write_bytes": wr * scale, "algorithmic_bytes_per_launch": alg,
         "duration_s_under_ncu": dur * dscale, "source": note}
path = os.path.join(ROOT, "profiles", "traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[workload] = entry
with open(path, "w") as f:
    json.dump(data, f, indent=1)
print(json.dumps(entry, indent=1))
