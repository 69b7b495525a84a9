"""Summarize .ncu-rep captures (ncu --set full) into a markdown table:
duration, DRAM bytes per launch, DRAM / SM / tensor-pipe utilization,
registers, achieved occupancy.  Usage: python tools/ncu_summary.py rep1 [rep2 ...]"""
import csv
import io
import subprocess
import sys

COLS = [
    ("dur us", "gpu__time_duration.sum", 1e-3),
    ("DRAM R MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM W MB", "dram__bytes_write.sum", 1e-6),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue %", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
]


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units = rd[0], rd[1]
    res = []
    for r in rd[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        vals = []
        for _, key, sc in COLS:
            k = next((h for h in hdr if h == key or h.endswith("." + key)), None)
            v = _num(d.get(k)) if k else None
            if v is not None and key == "gpu__time_duration.sum":
                unit = u.get(k, "")
                v = v * {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                         "msecond": 1e6}.get(unit, 1.0)  # -> ns
            if v is not None and key.startswith("dram__bytes"):
                unit = u.get(k, "")
                v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                         "GB": 1e9}.get(unit, 1)
            vals.append(None if v is None else v * sc)
        name = d.get("Kernel Name", "?").split("(")[0]
        res.append((name, vals))
    return res


print("| kernel | " + " | ".join(c[0] for c in COLS) + " |")
print("|---|" + "---|" * len(COLS))
for rep in sys.argv[1:]:
    for name, vals in rows_of(rep):
        cells = ["" if v is None else (f"{v:.1f}" if abs(v) < 1e5 else f"{v:.3g}") for v in vals]
        print(f"| `{name}` | " + " | ".join(cells) + " |")
