"""Summarise ncu outputs (launch lists and --set full reports) into profiles/ text files.

    python profiles/summarize.py launches <launches.csv>          # per-kernel time shares
    python profiles/summarize.py report <prof.ncu-rep>            # key metrics per launch
"""
import csv
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    d = OrderedDict()
    unit = ""
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0]
            d.setdefault(name, []).append(float(r["Metric Value"]))
            unit = r["Metric Unit"]
    tot = sum(sum(v) for v in d.values())
    out = [f"# ncu launch list {path}: gpu__time_duration.sum per launch (cold-cache, serialised)",
           f"{'kernel':60s} {'launches':>8s} {'avg_' + unit:>12s} {'share':>7s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v):12.2f} {sum(v) / tot:7.3f}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu --set full {path}"]
    for r in rows[2:]:
        out.append(f"## {r[hdr.index('Kernel Name')][:90]}")
        for k in KEYS:
            if k in hdr:
                out.append(f"  {k:62s} {r[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
        if "dram__bytes_read.sum" in hdr:
            def mb(k):
                v = float(r[hdr.index(k)].replace(",", ""))
                u = units[hdr.index(k)]
                return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            t = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            tu = units[hdr.index("gpu__time_duration.sum")]
            t_us = t * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(tu, 1.0)
            tot = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
            out.append(f"  => dram traffic {tot:.1f} MB per launch, {tot / t_us:.3f} TB/s over the launch")
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[2]) if sys.argv[1] == "launches" else report(sys.argv[2]))
