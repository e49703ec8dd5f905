"""Summarise ncu outputs into the markdown committed under profiles/.

    python tools/ncu_summary.py launches <launches.csv>       # per-kernel share of a launch list
    python tools/ncu_summary.py full <report.ncu-rep>         # key metrics per profiled launch
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", None),
    ("dram__bytes_write.sum", "dram_write_MB", None),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("smsp__inst_executed.sum", "warp_inst_M", 1e-6),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    print("| launch | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|---|" + "---:|" * len(KEYS))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = []
        for key, label, scale in KEYS:
            if key not in hdr:
                vals.append("-")
                continue
            v = r[hdr.index(key)].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                vals.append(v)
                continue
            u = units[hdr.index(key)]
            if scale is None:  # bytes -> MB, honouring the unit ncu chose
                mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                x *= mult
            elif key == "gpu__time_duration.sum":
                x *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            else:
                x *= scale
            vals.append(f"{x:.1f}")
        print(f"| {r[hdr.index('ID')]} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
