"""Time the DL conv2 kernels (and conv1, pool) on the full DL shapes
(BASELINE configs[4]: 16384^2 input -> 4096^2 x 8 conv2 input), 10 launches
each, CUDA events on one stream; compare every conv2 output to the FFMA one.

    python tools/conv2_variants.py [--h 16384] [--variants conv2_ffma,conv2_tc1,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, default=16384)
    ap.add_argument("--variants", default="conv2_ffma,conv2_tc1,conv2_tc4,conv2_tc5,conv2")
    ap.add_argument("--conv1", action="store_true", help="also time the conv1 variants")
    a = ap.parse_args()
    import torch
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    from paper_2012_09646_b200.programs import DeepLearning
    from paper_2012_09646_b200.programs.hits_dl import CONV2_TC5_SMEM, CONV2_TC_SMEM, CONV2_TC_THREADS, G2TC
    ctx = D.Context(device=0)
    p = DeepLearning(ctx, h=a.h, w=a.h)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    (h1, w1), (h2, w2), (h3, w3) = p.shapes
    st = torch.cuda.Stream()
    out = {}
    outs = {}

    def timeit(L, reps=10):
        L.raw(st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
            for _ in range(reps):
                L.raw(st.cuda_stream)
            e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    kb = p.kernel_bytes()
    for i, name in ((0, "conv1"), (2, "pool")) if a.conv1 else ():
        us = timeit(p.L[i])
        out[name] = {"us": us, "GBps": kb[name + "_x"] / us / 1e3}
    c1ref = p.t["c1x"].clone()
    L0 = p.L[0]
    for v in ("conv1_b3", "conv1_b4", "conv1_b4cs", "conv1_r2b3", "conv1_r2b3cs", "conv1_r2b2") if a.conv1 else ():
        for rows_per in ((8, 16, 24, 32) if "_r2" in v else (8, 16)):
            nrows = (h1 + 1) // 2 if "_r2" in v else h1  # the r2 kernels' grid.y walks row pairs
            g = (L0.grid.x, max(1, min(nrows, -(-rows_per * 148 // L0.grid.x))))
            L = ctx.prepare(v, g, 256, [p.a["x"], p.a["w1"], p.a["c1x"], a.h, a.h])
            us = timeit(L)
            torch.cuda.synchronize()
            out[f"{v}_r{rows_per}"] = {"us": us, "GBps": kb["conv1_x"] / us / 1e3,
                                      "same": bool(torch.equal(c1ref, p.t["c1x"]))}
    for v in a.variants.split(","):
        o = torch.full((h3 * w3 * 16,), -1.0, device="cuda")
        torch.cuda.synchronize()
        arr = ctx.register_tensor(f"c2_{v}", o)
        args = [p.a["px"], p.a["w2"], arr, h2, w2]
        if v == "conv2_ffma":
            L = ctx.prepare(v, ((w3 + 1) // 2 // 256 + 1, min(h3, 65535)), 256, args)
        elif v in ("conv2_tc1", "conv2_tc3"):
            L = ctx.prepare(v, 2 * 148, 128, args, smem=2 * 9 * 512 + 2 * 9 * 4096 + 64)
        elif v == "conv2_tman3x1":
            L = ctx.prepare(v, 148, 384, args, smem=1024 + 3 * 9 * 4096 + 3 * 9 * 4096 + 2 * 9 * 512 + 64)
        elif v == "conv2_tmar":
            from paper_2012_09646_b200.programs.hits_dl import CONV2_TMAR_SMEM, CONV2_TMAR_THREADS
            L = ctx.prepare(v, 148, CONV2_TMAR_THREADS, args, smem=CONV2_TMAR_SMEM)
        elif v.startswith("conv2_tmag") or v.startswith("conv2_tman"):  # (incl. conv2_tmanr1)
            from paper_2012_09646_b200.programs.hits_dl import CONV2_TMAG_SMEM
            L = ctx.prepare(v, 148, 256, args, smem=CONV2_TMAG_SMEM[int(v[-1])])
        elif v.startswith("conv2_tma"):
            from paper_2012_09646_b200.programs.hits_dl import CONV2_TMA_SMEM
            L = ctx.prepare(v, 148, 128, args, smem=CONV2_TMA_SMEM[int(v[-1])])
        elif v == "conv2_tc2":
            L = ctx.prepare(v, 2 * 148, 256, args, smem=2 * 9 * 512 + 2 * 9 * 4096 + 64)
        elif v == "conv2_tc5":
            L = ctx.prepare(v, 148, 384, args, smem=CONV2_TC5_SMEM)
        elif v == "conv2_tc4":
            L = ctx.prepare(v, G2TC, 128, args, smem=2 * 9 * 512 + 4 * 3 * 4 * 129 * 16 + 2 * 9 * 4096 + 64)
        elif v.startswith("conv2_ws") or v.startswith("conv2_rows") or v.startswith("conv2_h"):
            from paper_2012_09646_b200.programs.hits_dl import conv2_ws_launch
            th, sm = conv2_ws_launch(v)
            L = ctx.prepare(v, 148, th, args, smem=sm)
        elif v == "conv2":  # the product launch configuration (programs/hits_dl.py)
            from paper_2012_09646_b200.programs.hits_dl import CONV2_GRID, CONV2_SMEM, CONV2_THREADS
            L = ctx.prepare(v, CONV2_GRID, CONV2_THREADS, args, smem=CONV2_SMEM)
        else:
            L = ctx.prepare(v, G2TC, CONV2_TC_THREADS, args, smem=CONV2_TC_SMEM)
        us = timeit(L)
        torch.cuda.synchronize()
        outs[v] = o
        out[v] = {"us": us, "GBps": kb["conv2_x"] / us / 1e3}
    ref = outs.get("conv2_ffma")
    if ref is not None:
        for v, o in outs.items():
            d = (o - ref).abs()
            tol = 1e-4 * ref.abs() + 1e-4 * ref.pow(2).mean().sqrt()
            out[v]["bad_vs_ffma"] = int((d > tol).sum())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
