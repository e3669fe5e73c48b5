#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/ncu_summary.py gpurun_out/launches.csv [--only-bl] > profiles/...md
Per-launch ncu times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"(bl::k_\w+(<[^()]*>)?)", name)
    if m:
        return m.group(1)
    return name[:70]


def main():
    path = sys.argv[1]
    only = "--only-bl" in sys.argv
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        if only and not k.startswith("bl::"):
            continue
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0 if r["Metric Unit"] == "us" else 1e3)
        a = agg.setdefault(k, [0, 0.0, []])
        a[0] += 1
        a[1] += v
        a[2].append(v)
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total us | share | mean us | min us | max us |")
    print("|---|---|---|---|---|---|---|")
    for k, (c, t, vs) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t:.1f} | {100 * t / tot:.1f}% | {t / c:.2f} | {min(vs):.2f} | {max(vs):.2f} |")
    print(f"\ntotal kernel time {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")


if __name__ == "__main__":
    main()
