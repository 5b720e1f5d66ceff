"""Summarise ncu reports (.ncu-rep) and launch lists (.csv) for profiles/.

usage: python scripts/ncu_summary.py <out.md> <report-or-csv> [...]
Reads raw metrics with `ncu -i ... --page raw --csv` (works without a GPU).
"""
import collections
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time", "us", 1e-3),
    ("dram__bytes_read.sum", "DRAM read", "MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM write", "MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak", "%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak", "%", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %", "%", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %", "%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", "%", 1),
    ("launch__registers_per_thread", "regs/thread", "", 1),
    ("launch__grid_size", "grid", "", 1),
    ("launch__block_size", "block", "", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts", "", 1),
]


def unit_scale(v, unit):
    return v


def report_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
        for key, label, unit, _ in METRICS:
            if key in h:
                raw = r[h.index(key)].replace(",", "")
                u = units[h.index(key)]
                try:
                    v = float(raw)
                except ValueError:
                    continue
                # normalise to the label's unit
                if unit == "us":
                    v = v / 1e3 if u == "nsecond" else (v * 1e3 if u == "msecond" else v)
                elif unit == "MB":
                    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    v = v * scale
                d[label] = v
        res.append(d)
    return res


def launch_rows(path):
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    h = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            h = r
            continue
        if h is None or len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("stn::", "")
        name = name.replace("<unnamed>::", "")
        agg[name] += float(d["Metric Value"].replace(",", ""))
        cnt[name] += 1
    return agg, cnt


def main():
    out = sys.argv[1]
    lines = []
    for path in sys.argv[2:]:
        lines.append(f"## {os.path.basename(path)}\n")
        if path.endswith(".csv"):
            agg, cnt = launch_rows(path)
            tot = sum(agg.values())
            lines.append(f"{sum(cnt.values())} launches, {tot / 1e6:.3f} ms total "
                         "(ncu: serialised, cold-cache; compare shares)\n")
            lines.append("| kernel | launches | ms | share |\n|---|---|---|---|")
            for k, v in sorted(agg.items(), key=lambda x: -x[1]):
                lines.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / tot:.3f} |")
        else:
            rows = report_rows(path)
            labels = [m[1] for m in METRICS]
            lines.append("| kernel | " + " | ".join(labels) + " |")
            lines.append("|---" * (len(labels) + 1) + "|")
            for d in rows:
                name = d["kernel"].split("(")[0].replace("void ", "")[:60]
                vals = []
                for lab in labels:
                    v = d.get(lab)
                    vals.append("" if v is None else (f"{v:.1f}" if v < 1e4 else f"{v:.0f}"))
                lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
