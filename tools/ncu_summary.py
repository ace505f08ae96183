"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and,
optionally, a --set full report: per-kernel launches, mean time, share, and
for the full report DRAM bytes / throughput / SM and memory utilisation."""

import collections
import csv
import re
import subprocess
import sys


def kname(raw: str) -> str:
    raw = raw.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    m = re.match(r"(?:void\s+)?([\w:]+(?:<[^()]*?>)?)", raw)
    return m.group(1) if m else raw[:60]


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v,
             "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
        agg[kname(r[ki])].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean µs | share |", "|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {n} | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out)


def full(path: str) -> str:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    ki = hdr.index("Kernel Name")
    out = ["| kernel | time | DRAM read | DRAM write | DRAM % peak | SM % | regs | warps active % |",
           "|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        g = lambda w: r[idx[w]] if w in idx else "-"  # noqa: E731
        out.append(f"| {kname(r[ki])} | {g('gpu__time_duration.sum')} | "
                   f"{g('dram__bytes_read.sum')} | {g('dram__bytes_write.sum')} | "
                   f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{g('launch__registers_per_thread')} | "
                   f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} |")
    units = rows[1]
    out.append("")
    out.append("units: " + ", ".join(f"{w}={units[i]}" for w, i in idx.items()))
    return "\n".join(out)


def traffic(path: str) -> dict:
    """Mean DRAM bytes (read + write) per launch per kernel of a --set full
    report: the `roofline.traffic` figure bench.py reports."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = collections.defaultdict(list)
    for r in rows[2:]:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        acc[kname(r[ki]).split("<")[0]].append(b)
    return {k: sum(v) / len(v) for k, v in acc.items()}


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        import json
        print(json.dumps({"report": sys.argv[2], "note": sys.argv[3] if len(sys.argv) > 3 else "",
                          "dram_bytes_per_launch": traffic(sys.argv[2])}, indent=1))
        sys.exit(0)
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print()
        print(full(sys.argv[2]))
