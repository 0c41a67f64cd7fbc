"""MMUL lab (BASELINE configs[3] ML, 10M x 200 -> 10 classes): the product
nb_mmul / rr_mmul against other forms registered as <kernel>_<variant>
(measured once: *_ws, the feature halves split across warps so weight loads
are single-address broadcasts -- 1.77 / 1.83 vs 1.59 / 1.58 ms, removed;
profiles/r2_mmul_ws_lab.json);
ms per launch (CUDA events, 5 launches after 1, one stream), HBM fraction of
the algorithmic 4F + 4C bytes per row, outputs compared bitwise.

    python tools/mmul_lab.py [--variants ws] [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--variants", default="")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    peak = float(bench.load_peaks()[0].get("hbm_gbs", 6548.0))
    ctx = D.Context(device=0)
    p = bench.make_program("ml", ctx, "resident")
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    base = {L.kernel.name: L for L in p.launch_sequence() if L.kernel.name in ("nb_mmul", "rr_mmul")}
    st = torch.cuda.Stream()
    res = {}
    for kind, L0 in base.items():
        outn = "r1" if kind == "nb_mmul" else "r2"
        ref = None
        confs = [(kind, L0.block.x, L0.grid.x)] + [(kind, 64, g) for g in (296, 444)] + \
                [(f"{kind}_{v}", L0.block.x, L0.grid.x) for v in args.variants.split(",") if v]
        for name, blk, grd in confs:
            L = ctx.prepare(name, grd, blk, list(L0.args_in) if hasattr(L0, "args_in") else
                            [p.a["X"], p.a["theta"], p.a["prior"], p.a["r1"], p.n, p.f, p.c] if kind == "nb_mmul" else
                            [p.a["Z"], p.a["W"], p.a["r2"], p.n, p.f, p.c], L0.smem)
            L.raw(st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record()
                for _ in range(5):
                    L.raw(st.cuda_stream)
                e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 5
            y = p.t[outn].clone()
            if ref is None:
                ref = y
            byts = (4.0 * p.f + 4.0 * p.c) * p.n
            r = {"ms": round(ms, 4), "hbm_frac": round(byts / (ms * 1e-3) / 1e9 / peak, 3),
                 "bitwise_same_as_product": bool(torch.equal(ref, y))}
            r.update({"block": blk, "grid": grd})
            res[f"{name}_b{blk}_g{grd}"] = r
            print(name, json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
