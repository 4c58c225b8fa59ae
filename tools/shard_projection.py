#!/usr/bin/env python
"""Multi-GPU projection on ONE GPU: time every LPT shard of the N-GPU VGG16 step alone.

    python tools/shard_projection.py [--steps 10] [--out profiles/r02_shard_projection.json]

For N in (2, 4, 8) and every rank k, `bench.py --emulate-world N --emulate-rank k` runs exactly the work rank k does in
the N-GPU job (its layers, its global factor tags, its StreamedStep groups), without the collective, on this GPU.  The
N-GPU step is at least max_k t_k; the projected speed-up is t_1 / (max_k t_k + t_allgather), where t_allgather is the
all-gather of the packed preconditioned gradients, NOT measured here (one GPU) and reported separately as an estimate
at an assumed NVSwitch all-gather bus bandwidth.  Each shard runs alone, so it sees the whole GPU, as it would on its
own B200.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(extra, steps, workload):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(steps), "--warmup", "3",
           "--no-cpu-baseline", "--workload", workload, *extra]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--busbw-gbs", type=float, default=700.0, help="assumed all-gather bus bandwidth (not measured)")
    ap.add_argument("--workload", default="vgg16")
    ap.add_argument("--overlap", action="store_true", help="shards with the opt-in overlapped power iteration")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.out is None:
        sfx = ("" if args.workload == "vgg16" else "_" + args.workload) + ("_overlap" if args.overlap else "")
        args.out = os.path.join(ROOT, "profiles", f"r02_shard_projection{sfx}.json")
    import bench
    from paper_2206_15397_b200.partition import layer_cost, lpt_partition

    layers, _, _, r, p = bench.WORKLOADS[args.workload][:5]
    ov = ["--overlap"] if args.overlap else []
    one = run(ov, args.steps, args.workload)
    t1 = one["ms_per_step"]
    res = {"workload": args.workload, "overlapped_power_iteration": bool(args.overlap), "t1_ms": t1, "t1_line": {k: one[k] for k in ("ms_per_step", "stage_ms", "clocks")}, "worlds": {}}
    costs = [layer_cost(a, g, r, p) for a, g in layers]
    for N in (int(x) for x in args.worlds.split(",")):
        parts = lpt_partition(costs, N)
        shards = []
        for k in range(N):
            if not parts[k]:
                shards.append({"rank": k, "layers": [], "ms": 0.0})
                continue
            ln = run(["--emulate-world", str(N), "--emulate-rank", str(k)] + ov, args.steps, args.workload)
            shards.append({"rank": k, "layers": parts[k], "ms": ln["ms_per_step"], "stage_ms": ln["stage_ms"]})
            print(f"N={N} rank {k} layers {parts[k]}: {ln['ms_per_step']:.3f} ms", flush=True)
        tmax = max(s["ms"] for s in shards)
        # all-gather of the packed gradients: every rank contributes its padded chunk (GatherLayout)
        sizes = [a * g for a, g in layers]
        chunk = max(sum(sizes[l] for l in part) for part in parts) * 4
        ag_ms = (N - 1) * chunk / (args.busbw_gbs * 1e9) * 1e3
        res["worlds"][N] = {"shards": shards, "max_shard_ms": tmax, "allgather_bytes_per_rank": chunk,
                            "allgather_ms_estimate": ag_ms,
                            "projected_speedup_compute_only": t1 / tmax,
                            "projected_speedup_with_allgather_estimate": t1 / (tmax + ag_ms)}
        print(f"N={N}: max shard {tmax:.3f} ms -> {t1 / tmax:.2f}x (with all-gather estimate {t1 / (tmax + ag_ms):.2f}x)",
              flush=True)
    res["note"] = (f"all-gather time is an estimate at an ASSUMED {args.busbw_gbs} GB/s bus bandwidth "
                   "((N-1) x padded chunk / busbw); shards measured alone on one B200 with bench.py --emulate-world")
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
