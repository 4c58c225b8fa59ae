"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

    python tools/launches.py launches.csv [--last N]

Prints per-kernel totals (us, count, grid) over the last N launches (default: all) and the launch sequence.
"""
import argparse
import collections
import csv
import re


def short(name):
    name = re.sub(r"\(.*", "", name)
    for junk in ("rkfac_b200::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::", "void "):
        name = name.replace(junk, "")
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", type=int, default=0)
    ap.add_argument("--seq", action="store_true")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10 and r[0].isdigit()]
    if a.last:
        rows = rows[-a.last:]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        t = float(r[-1]) / 1e3
        tot += t
        e = agg.setdefault(f"{short(r[4])} grid{r[8]}", [0, 0.0])
        e[0] += 1
        e[1] += t
    print(f"{len(rows)} launches, {tot:.1f} us total (serialised, cold-cache)")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t:9.1f} us {100 * t / tot:5.1f}%  {c:3d}x  {k}")
    if a.seq:
        for r in rows:
            print(f"{float(r[-1]) / 1e3:8.1f}  {short(r[4])} grid{r[8]}")


if __name__ == "__main__":
    main()
