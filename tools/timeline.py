#!/usr/bin/env python
"""Summarise the concurrent kernel timeline of one step (bench.py --trace out.json, a chrome trace from CUPTI).

Prints, per stream, the busy time and the kernel sequence with start offsets, the number of CTAs resident over time
(sum of grid sizes of overlapping kernels, a proxy for SM fill) and the critical stream.
usage: python tools/timeline.py trace.json [--list STREAM] [--bins N]
"""
import argparse
import collections
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--list", type=int, default=-1, help="print every kernel of this stream")
    ap.add_argument("--bins", type=int, default=40)
    args = ap.parse_args()
    ev = json.load(open(args.trace))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and e.get("ph") == "X"]
    t0 = min(e["ts"] for e in ks)
    t1 = max(e["ts"] + e["dur"] for e in ks)
    print(f"{len(ks)} device activities, span {(t1 - t0) / 1e3:.3f} ms")
    by = collections.defaultdict(list)
    for e in ks:
        by[e["args"].get("stream", e.get("tid"))].append(e)
    for st, es in sorted(by.items(), key=lambda kv: -sum(e["dur"] for e in kv[1])):
        es.sort(key=lambda e: e["ts"])
        busy = sum(e["dur"] for e in es)
        first, last = es[0]["ts"] - t0, es[-1]["ts"] + es[-1]["dur"] - t0
        agg = collections.Counter()
        for e in es:
            agg[e["name"].split("(")[0][:40]] += e["dur"]
        top = ", ".join(f"{k} {v / 1e3:.2f}" for k, v in agg.most_common(5))
        print(f"stream {st}: {len(es)} acts, busy {busy / 1e3:.3f} ms, {first / 1e3:.3f} -> {last / 1e3:.3f} ms | {top}")
        if st == args.list:
            for e in es:
                g = e["args"].get("grid", "")
                print(f"   {(e['ts'] - t0) / 1e3:8.3f} +{e['dur'] / 1e3:7.3f}  {str(g):>14}  {e['name'][:60]}")
    # CTA fill over time
    nb = args.bins
    w = (t1 - t0) / nb
    fill = [0.0] * nb
    for e in ks:
        g = e["args"].get("grid")
        if not g:
            continue
        ctas = g[0] * g[1] * g[2]
        a, b = e["ts"] - t0, e["ts"] + e["dur"] - t0
        for i in range(int(a // w), min(nb - 1, int(b // w)) + 1):
            lo, hi = max(a, i * w), min(b, (i + 1) * w)
            if hi > lo:
                fill[i] += ctas * (hi - lo) / w
    print("resident CTAs (grid sum) per time bin of %.3f ms:" % (w / 1e3))
    print(" ".join(f"{x:.0f}" for x in fill))


if __name__ == "__main__":
    main()
