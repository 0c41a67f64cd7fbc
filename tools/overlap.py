"""Schedule evidence: run one benchmark DAG with the scheduler's timeline on
and compute the paper's overlap metrics (§V-F):
  CT  = fraction of kernel time overlapping any transfer
  TC  = fraction of transfer time overlapping any kernel
  CC  = fraction of kernel time overlapping other kernels
  TOT = fraction of all item time overlapping any other item
    python tools/overlap.py --bench bs --mode stream [--runs 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def covered(a, b, u):
    """Length of [a,b] covered by the union intervals u."""
    s = 0.0
    for x, y in u:
        lo, hi = max(a, x), min(b, y)
        if hi > lo:
            s += hi - lo
    return s


def metrics(items):
    K = [(r[5], r[6]) for r in items if r[0] == "kernel"]
    T = [(r[5], r[6]) for r in items if r[0] != "kernel"]
    uT = union(T)
    uK = union(K)
    kt = sum(b - a for a, b in K)
    tt = sum(b - a for a, b in T)
    ct = sum(covered(a, b, uT) for a, b in K) / kt if kt else 0.0
    tc = sum(covered(a, b, uK) for a, b in T) / tt if tt else 0.0
    cc_num = 0.0
    for i, (a, b) in enumerate(K):
        cc_num += covered(a, b, union(K[:i] + K[i + 1:]))
    cc = cc_num / kt if kt else 0.0
    allv = K + T
    tot_num = 0.0
    for i, (a, b) in enumerate(allv):
        tot_num += covered(a, b, union(allv[:i] + allv[i + 1:]))
    tot = tot_num / (kt + tt) if (kt + tt) else 0.0
    span = (max(b for _, b in allv) - min(a for a, _ in allv)) if allv else 0.0
    return {"CT": ct, "TC": tc, "CC": cc, "TOT": tot, "kernel_ms": kt, "transfer_ms": tt,
            "span_ms": span, "items": len(allv)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default="bs")
    ap.add_argument("--mode", default="stream")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import bench
    from paper_2012_09646_b200 import dagrt as D
    res = {}
    for policy in ("parallel", "serial"):
        ctx = D.Context(device=0, policy=policy)
        p = bench.make_program(args.bench, ctx, args.mode)
        p.load_inputs(0)
        p.run()
        ctx.timeline(True)
        for _ in range(args.runs):
            p.run()
        items = ctx.timeline_export()
        ctx.timeline(False)
        m = metrics(items)
        m["span_ms"] /= args.runs
        res[policy] = m
        if policy == "parallel":
            res["timeline"] = [list(r) for r in items[: 400]]
        ctx.close()
        del p
    out = {"bench": args.bench, "mode": args.mode, **res}
    s = json.dumps(out)
    if args.out:
        open(args.out, "w").write(s)
    print(json.dumps({k: v for k, v in out.items() if k != "timeline"}, indent=1))


if __name__ == "__main__":
    main()
