"""Time the ML MMUL kernels on the full ML shapes (BASELINE configs[3]:
10M x 200) with two (128-thread CTAs, the product) and four (256-thread
CTAs) threads per row; compare their outputs.  (The four-per-row path was measured slower and removed; the tool now times the product only.)

    python tools/mmul_variants.py [--n 10000000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    a = ap.parse_args()
    import torch
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200.programs import MLEnsemble
    ctx = D.Context(device=0)
    p = MLEnsemble(ctx, n=a.n)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    n, f, c = p.n, p.f, p.c
    st = torch.cuda.Stream()
    out = {}

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

    res = {}
    for threads in (128,):
        rows = 64
        gm = max(1, min(-(-n // rows), 2 * 148))
        smem = 4 * c * f + 16 + 2 * rows * 4 * f
        for name, args in (("nb_mmul", [p.a["X"], p.a["theta"], p.a["prior"]]), ("rr_mmul", [p.a["Z"], p.a["W"]])):
            o = torch.zeros(n * c, device="cuda")
            torch.cuda.synchronize()
            arr = ctx.register_tensor(f"mm_{name}_{threads}", o)
            L = ctx.prepare(name, gm, threads, args + [arr, n, f, c], smem=smem)
            us = timeit(L)
            torch.cuda.synchronize()
            res[(name, threads)] = o
            out[f"{name}_t{threads}"] = {"us": us, "GBps": (4 * n * f + 4 * n * c) / us / 1e3}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
