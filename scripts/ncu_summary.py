"""Summarise ncu outputs pulled back by gpurun.

  python scripts/ncu_summary.py launches <launches.csv>   per-kernel count / time / share
  python scripts/ncu_summary.py full <report.ncu-rep>      key metrics per captured launch
"""
import collections
import csv
import io
import subprocess
import sys


def _csv_rows(text):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def launches(path):
    rows = _csv_rows(open(path).read())
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        n = r["Kernel Name"].split("(")[0].replace("msb::", "")
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'total_us':>11s} {'us/launch':>10s} {'share':>6s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:34s} {c:8d} {t:11.1f} {t / c:10.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':34s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rdr = list(csv.reader(io.StringIO(out)))
    h, units = rdr[0], rdr[1]
    for row in rdr[2:]:
        name = row[h.index("Kernel Name")].split("(")[0]
        print(f"== {name}")
        for m in FULL:
            if m in h:
                i = h.index(m)
                print(f"   {m:58s} {row[i]:>14s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
