"""conv1 lab (BASELINE configs[4] DL, 16384^2 fp32 input -> 8192^2 x 8):
the product conv1 against the cp.async-staged banded variants (exp
conv1_ca<PFP>b<CTAs/SM>, csrc/conv1.cuh conv1_body3) for two band counts;
us per launch (CUDA events, 10 launches after 2), HBM fraction of the
algorithmic 4 B/input + 32 B/output pixel, output compared bitwise with the
product's; then ragged shapes (odd H/W, W % 4 != 0, tiny) bitwise.

    python tools/conv1_variants.py [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SMEM = {"ca1": 9 * 4112, "ca2": 13 * 4112}


def smem_of(name):
    for k, v in SMEM.items():
        if name.startswith("conv1_" + k):
            return v
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--variants", default="conv1_ca1b4,conv1_ca1b3,conv1_ca2b3,conv1_ca2b4,conv1_ca2b4cs")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()
    peak = float(bench.load_peaks()[0].get("hbm_gbs", 6548.0))
    ctx = D.Context(device=0)
    p = bench.make_program("dl", ctx, "resident")
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, h, w = p.a, p.h, p.w
    (h1, w1), _, _ = p.shapes
    byts = 4.0 * h * w + 32.0 * h1 * w1
    L0 = p.L[0]
    st = torch.cuda.Stream()
    res, ref = {}, None
    for name in ["conv1"] + args.variants.split(","):
        for gy in ([L0.grid.y] if name == "conv1" else [148, 296, 592]):
            L = ctx.prepare(name, (L0.grid.x, gy), 256, [a["x"], a["w1"], a["c1x"], h, w], smem_of(name))
            for _ in range(2):
                L.raw(st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record()
                for _ in range(10):
                    L.raw(st.cuda_stream)
                e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / 10 * 1e3
            y = p.t["c1x"].clone()
            if ref is None:
                ref = y
            r = {"grid_y": gy, "us": round(us, 1), "hbm_frac": round(byts / (us * 1e-6) / 1e9 / peak, 3),
                 "bitwise_same_as_product": bool(torch.equal(ref, y))}
            res[f"{name}_gy{gy}"] = r
            print(name, json.dumps(r), flush=True)
            del y
    del ref
    shapes = [(33, 35), (64, 1000), (1, 1), (3, 5), (130, 1030), (7, 4100), (517, 2051)]
    for v in args.variants.split(","):
        ok = True
        for (hh, ww) in shapes:
            hh1, ww1 = (hh + 1) // 2, (ww + 1) // 2
            x = torch.rand(hh * ww + 3, device="cuda")
            xs = x[1:1 + hh * ww] if ww % 4 else x[:hh * ww]
            wt = torch.randn(72, device="cuda")
            outs = []
            for name in ("conv1", v):
                y = torch.full((hh1 * ww1 * 8,), -7.0, device="cuda")
                c2 = D.Context(device=0)
                X, Wt, Y = (c2.register_tensor(k, tt) for k, tt in (("x", xs), ("w", wt), ("y", y)))
                gx = max(1, -(-((ww1 + 1) // 2) // 256))
                gy = max(1, min((hh1 + 1) // 2, 148))
                c2.launch(name, (gx, gy), 256, X, Wt, Y, hh, ww, smem=smem_of(name))
                c2.sync()
                c2.close()
                outs.append(y.clone())
            ok = ok and bool(torch.equal(outs[0], outs[1]))
        res[f"ragged_{v}"] = ok
        print("ragged", v, ok, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
