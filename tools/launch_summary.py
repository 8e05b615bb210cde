"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel template.

usage: python tools/launch_summary.py launches.csv > summary.md
Only this library's kernels (namespace tzcdev) are counted in the shares.
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [l for l in open(path) if not l.startswith("==")]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in csv.DictReader(rows):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if "tzcdev::" not in name:
            continue
        us = float(r["Metric Value"]) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        if r["Metric Unit"] == "msecond":
            us = float(r["Metric Value"]) * 1000.0
        elif r["Metric Unit"] == "usecond":
            us = float(r["Metric Value"])
        tot[name] += us
        cnt[name] += 1
    all_us = sum(tot.values())
    print("| kernel (template) | launches | total us | us / launch | share of our kernels |")
    print("|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {100 * tot[k] / all_us:.1f}% |")
    print(f"\nTotal of our kernels: {all_us:.1f} us over {sum(cnt.values())} launches.")


if __name__ == "__main__":
    main(sys.argv[1])
