"""Per-stage DL parity report for one conv2 variant (debug aid).

    python tools/dl_debug.py [--variant conv2|conv2_tc1|conv2_ffma] [--sizes 64x64,515x517]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import dl as odl  # noqa: E402
from paper_2012_09646_b200 import dagrt as D  # noqa: E402

D.load_experimental()  # conv1/conv2 variants live in libdagrt_exp.so
from paper_2012_09646_b200.programs import DeepLearning  # noqa: E402
from paper_2012_09646_b200.programs.hits_dl import G2TC  # noqa: E402


def close(g, o, rel=1e-4):
    o = np.asarray(o, np.float64)
    g = np.asarray(g, np.float64)
    rms = np.sqrt(np.mean(o * o)) if o.size else 0.0
    bad = np.abs(g - o) > rel * np.abs(o) + rel * rms
    return int(bad.sum()), (np.argwhere(bad)[:5].tolist() if bad.any() else [])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="conv2")
    ap.add_argument("--sizes", default="19x23,64x64,515x517")
    ap.add_argument("--serial", action="store_true")
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    for s in a.sizes.split(","):
        h, w = map(int, s.split("x"))
        ctx = D.Context(device=0, policy="serial" if a.serial else "parallel")
        p = DeepLearning(ctx, h=h, w=w)
        (h1, w1s), (h2, w2s), (h3, w3s) = p.shapes
        if a.variant != "conv2":
            for i, b in ((4, "x"), (5, "y")):
                L = p.L[i]
                args = [p.a[f"p{b}"], p.a["w2"], p.a[f"c2{b}"], h2, w2s]
                if a.variant == "conv2_ffma":
                    p.L[i] = ctx.prepare(a.variant, ((w3s + 1) // 2 // 256 + 1, h3), 256, args)
                elif a.variant == "conv2_tc1":
                    p.L[i] = ctx.prepare(a.variant, 2 * G2TC, 128, args, smem=2 * 9 * 512 + 2 * 9 * 4096 + 64)
        p._batch = p._steps = None  # the launch list was edited in place
        p.load_inputs(0)
        if a.trace:
            import torch
            p.run()
            ctx.sync()
            names = ["c1x", "c1y", "px", "py", "c2x", "c2y", "z"]
            p.begin_run()
            for i, L in enumerate(p.L):
                before = {n: p.t[n].clone() for n in names}
                L()
                ctx.sync()
                torch.cuda.synchronize()
                changed = [n for n in names if not torch.equal(before[n], p.t[n])]
                print("  launch", i, L.kernel.name, "changed", changed, flush=True)
            p.end_run()
        else:
            p.run()
        ctx.sync()
        spec = synth.spec_dl(h, w)
        x = synth.draw(p.seed, "x", spec["x"]).reshape(h, w)
        y = synth.draw(p.seed, "y", spec["y"]).reshape(h, w)
        w1 = synth.draw(p.seed, "w1", spec["w1"])
        w2 = synth.draw(p.seed, "w2", spec["w2"])
        wd = synth.draw(p.seed, "wd", spec["wd"])
        o = odl.dl(x, y, w1, w2, wd)
        rep = []
        for name, shp in (("c1x", (h1, w1s, 8)), ("c1y", (h1, w1s, 8)), ("px", (h2, w2s, 8)),
                          ("py", (h2, w2s, 8)), ("c2x", (h3, w3s, 16)), ("c2y", (h3, w3s, 16))):
            if np.prod(shp) == 0:
                continue
            got = p.t[name][:int(np.prod(shp))].cpu().numpy().reshape(shp)
            rep.append((name, close(got, o[name])))
        print(a.variant, s, rep, flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
