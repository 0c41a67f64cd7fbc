"""IMG stencil lab (BASELINE configs[2], 16384^2 fp32): the product blur /
sobel against the staging variants (exp blur_pf<N> / sobel_pf<N>: N input
rows of global loads in flight per thread in registers; blur_ca<N> /
sobel_ca<N>: cp.async into a ring of N + 1 shared rows) and rows per CTA
(grid.y); us per launch (CUDA events, 10 launches after 2, one stream),
HBM fraction of the algorithmic 8 B/pixel, output compared bitwise with the
product's.  Then the whole IMG DAG (resident) with the stencil vertices
swapped for the best variant.

    python tools/img_variants.py [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--variants", default="pf2,ca2,ca3,ca4,ca6")
    ap.add_argument("--rows", default="64,128")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200.programs.img_ml import IMG_BLUR_L, IMG_COLS, IMG_THREADS
    D.load_experimental()
    peak = float(bench.load_peaks()[0].get("hbm_gbs", 6548.0))
    ctx = D.Context(device=0)
    p = bench.make_program("img", ctx, "resident")
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, h, w = p.a, p.h, p.w
    st = torch.cuda.Stream()
    res = {}
    refs = {}
    for kind in ("blur", "sobel"):
        for name in [kind] + [f"{kind}_{v}" for v in args.variants.split(",")]:
            for rows in [int(x) for x in args.rows.split(",")]:
                grid = (max(1, -(-w // IMG_COLS)), max(1, -(-h // rows)))
                if kind == "blur":
                    L = ctx.prepare(name, grid, IMG_THREADS, [a["img"], a["bl"], h, w, IMG_BLUR_L[0], IMG_BLUR_L[1]])
                    outn = "bl"
                else:
                    L = ctx.prepare(name, grid, IMG_THREADS, [a["bs"], a["ms"], h, w])
                    outn = "ms"
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
                y = p.t[outn].clone()
                if kind not in refs:
                    refs[kind] = y
                r = {"us": round(us, 1), "hbm_frac": round(8.0 * h * w / (us * 1e-6) / 1e9 / peak, 3),
                     "bitwise_same_as_product": bool(torch.equal(refs[kind], y))}
                res[f"{name}_rows{rows}"] = r
                print(name, rows, json.dumps(r), flush=True)
                del y
    # ragged shapes (W % 4 != 0, tiny images, partial tiles): bitwise against the product
    shapes = [(515, 517), (64, 1000), (1, 1), (3, 5), (130, 1030), (7, 4096)]
    for kind in ("blur", "sobel"):
        for v in args.variants.split(","):
            ok = True
            for (hh, ww) in shapes:
                x = torch.rand(hh * ww + 3, device="cuda")
                xs = x[1:1 + hh * ww] if ww % 4 else x[:hh * ww]  # misaligned source when W is ragged
                outs = []
                for name in (kind, f"{kind}_{v}"):
                    y = torch.full((hh * ww,), -7.0, device="cuda")
                    c2 = D.Context(device=0)
                    X = c2.register_tensor("x", xs)
                    Y = c2.register_tensor("y", y)
                    grid = (max(1, -(-ww // IMG_COLS)), max(1, -(-hh // 64)))
                    extra = [IMG_BLUR_L[0], IMG_BLUR_L[1]] if kind == "blur" else []
                    c2.launch(name, grid, IMG_THREADS, X, Y, hh, ww, *extra)
                    c2.sync()
                    c2.close()
                    outs.append(y.clone())
                ok = ok and bool(torch.equal(outs[0], outs[1]))
            res[f"ragged_{kind}_{v}"] = ok
            print("ragged", kind, v, ok, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
