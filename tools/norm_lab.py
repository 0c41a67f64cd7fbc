"""NORM lab (BASELINE configs[3] ML, 10M x 200 int32): the product k_norm
with its dynamic shared memory varied -- the register path (below two ring
chunks) against the cp.async.bulk ring with 3 / 4 / 6 chunks of 2 RL rows
in flight; ms per launch (CUDA events, 3 launches after 1), HBM fraction of
the algorithmic 12 B/element, Z compared bitwise across configurations.

    python tools/norm_lab.py [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--smem", default="48000,64000,96000")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200.programs.img_ml import NORM_GRID, NORM_THREADS
    peak = float(bench.load_peaks()[0].get("hbm_gbs", 6548.0))
    ctx = D.Context(device=0)
    p = bench.make_program("ml", ctx, "resident")
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, n, f = p.a, p.n, p.f
    res, ref = {}, None
    for sm in [int(x) for x in args.smem.split(",")]:
        L = ctx.prepare("norm", NORM_GRID, NORM_THREADS, [a["X"], a["Z"], a["stats"], n, f], sm)
        L()
        ctx.sync()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(3):
            e0.record()
            L()
            ctx.sync()
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        z = p.t["Z"].clone()
        if ref is None:
            ref = z
        m = min(ms)
        r = {"smem": sm, "ms": round(m, 4), "hbm_frac": round(12.0 * n * f / (m * 1e-3) / 1e9 / peak, 3),
             "bitwise_same_as_first": bool(torch.equal(ref, z))}
        res[str(sm)] = r
        print(json.dumps(r), flush=True)
        del z
    if args.out:
        with open(args.out, "w") as fo:
            json.dump(res, fo, indent=1)


if __name__ == "__main__":
    main()
