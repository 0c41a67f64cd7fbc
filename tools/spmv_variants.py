"""Time the padded non-zero-split SpMV kernels (product "spmv" and its
experimental variants) on the HITS graph (BASELINE configs[4]): y = A^T h and
y = A a with the program's own plans and arrays, 10 launch pairs per grid
size, CUDA events on one stream; results compared with the product's.

    python tools/spmv_variants.py [name,name,...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    from paper_2012_09646_b200.programs import Hits
    from paper_2012_09646_b200.programs.hits_dl import SPMV_WARPS
    ctx = D.Context(device=0)
    p = Hits(ctx)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, n = p.a, p.n
    cap = (p.a["a2"].nbytes - 4 * n - 16) // (12 * SPMV_WARPS)  # largest grid the workspace holds
    st = torch.cuda.Stream()
    out, ref = {}, None
    sel = sys.argv[1].split(",") if len(sys.argv) > 1 else None
    for name in ("spmv", "spmv_pad", "spmv_tma4", "spmv_tma8"):
        if sel and name not in sel:
            continue
        for grid in (148 * 4, 148 * 8, 148 * 12, 148 * 16):
            if grid > cap:
                continue
            Ls = [ctx.prepare(name, grid, 256, [a["rpt"], a["cit"], a["plant"], a["h1"], a["a2"], n]),
                  ctx.prepare(name, grid, 256, [a["rp"], a["ci"], a["plan"], a["a1"], a["h2"], n])]
            for _ in range(2):
                for L in Ls:
                    L.raw(st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record()
                for _ in range(10):
                    for L in Ls:
                        L.raw(st.cuda_stream)
                e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            y = p.vec("a2").clone()
            if ref is None:
                ref = y
            out[f"{name}_g{grid}"] = {"us_per_launch": us, "bitwise_same_as_first": bool(torch.equal(ref, y)),
                                      "max_rel_diff": float(((y - ref).abs() / ref.abs().clamp_min(1e-30)).max())}
            print(name, grid, round(us, 1), flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
