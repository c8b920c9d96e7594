#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
shares of the captured launches (cold-cache, serialised: compare SHARES, not absolutes).
  python tools/launch_summary.py profiles/rNN_launches_n1.csv profiles/rNN_launches_n1_summary.txt "<command>"
"""
import csv
import sys
from collections import defaultdict


def main(src, dst, cmd=""):
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        if "phase_gate_kernel" in name:  # the phase pass's host-issue hold, not step work
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    out = [f"launch list: {cmd}", f"total {total:.1f} us over {sum(cnt.values())} launches"]
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"{t / total:6.3f}  n={cnt[name]:3d}  avg={t / cnt[name]:8.2f} us  {name}")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:12]))


if __name__ == "__main__":
    main(*sys.argv[1:4])
