"""Write profiles/roofline_traffic.json from an `ncu --set full` report: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) and duration per launch, averaged per
kernel name.  bench.py reads it to fill roofline.traffic (ncu replays are cold-cache:
the bytes include compulsory misses that a warm in-graph launch may hit in L2).

usage: python scripts/traffic_from_ncu.py [--units KERNEL=N ...] <report.ncu-rep> [...]
  --units k_sweep_ws=12: the captured launch of KERNEL processed N units (the persistent
  sweep kernel runs a chunk of sweeps per launch); dram_bytes/duration are also given per
  unit ("per_unit").
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("msb::", "")
        def val(m):
            i = h.index(m)
            return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        a = res.setdefault(name, dict(launches=0, dram_bytes=0.0, duration_us=0.0))
        a["launches"] += 1
        a["dram_bytes"] += val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        a["duration_us"] += val("gpu__time_duration.sum")
    for a in res.values():
        a["dram_bytes"] /= a["launches"]
        a["duration_us"] /= a["launches"]
    return res


if __name__ == "__main__":
    allk = {}
    units = {}
    args = sys.argv[1:]
    paths = []
    while args:
        a = args.pop(0)
        if a == "--units":
            k, n = args.pop(0).split("=")
            units[k] = int(n)
        else:
            paths.append(a)
    for p in paths:
        allk.update(read(p))
    for name, a in allk.items():
        for k, n in units.items():
            if name.startswith(k):
                a["units_per_launch"] = n
                a["per_unit"] = {"dram_bytes": a["dram_bytes"] / n,
                                 "duration_us": a["duration_us"] / n}
    doc = {"source": [os.path.relpath(p, ROOT) for p in paths],
           "note": "ncu --set full --clock-control none, cold cache per replay; per-launch means",
           "kernels": allk}
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    json.dump(doc, open(path, "w"), indent=1)
    print(json.dumps(doc, indent=1))
