"""Time the SpMV L2-policy variants (same arithmetic, bit-identical results)
on the HITS graph (BASELINE configs[4]): y = A^T h and y = A a, 20 launches
each, CUDA events on one stream.

    python tools/spmv_variants.py
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
    ctx = D.Context(device=0)
    p = Hits(ctx)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a = p.a
    n = p.n
    from paper_2012_09646_b200.programs.hits_dl import spmv_out_bytes
    _, grid = spmv_out_bytes(n, p.e)
    st = torch.cuda.Stream()
    out = {}
    ref = None
    from paper_2012_09646_b200.programs.hits_dl import spmv_plan
    plan, pg, ws = spmv_plan(p.csr[0])
    plant, pgt, wst = spmv_plan(p.csr[2])
    a = dict(a)
    a["plan"] = ctx.register_tensor("plan", torch.from_numpy(plan).cuda())
    a["plant"] = ctx.register_tensor("plant", torch.from_numpy(plant).cuda())
    # the plan kernel's workspace (chunk sums) is larger than merge-path's: own outputs
    ya = torch.zeros((4 * n + max(ws, wst)) // 4 + 1, device="cuda")
    yh = torch.zeros_like(ya)
    a["a2p"] = ctx.register_tensor("a2p", ya)
    a["h2p"] = ctx.register_tensor("h2p", yh)
    for name in ("spmv", "spmv_plan", "spmv_as1", "spmv_sync", "spmv_x0s1", "spmv_x1s1"):
        if name == "spmv_plan":  # row-class kernel (alternative; needs the plan workspace in y)
            Ls = [ctx.prepare(name, pgt, 256, [a["rpt"], a["cit"], a["plant"], a["h1"], a["a2p"], n]),
                  ctx.prepare(name, pg, 256, [a["rp"], a["ci"], a["plan"], a["a1"], a["h2p"], n])]
        else:
            Ls = [ctx.prepare(name, grid, 256, [a["rpt"], a["cit"], a["h1"], a["a2"], n]),
                  ctx.prepare(name, grid, 256, [a["rp"], a["ci"], a["a1"], a["h2"], n])]
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
        y = ya[:n].clone() if name == "spmv_plan" else p.vec("a2").clone()
        if ref is None:
            ref = y
        out[name] = {"us_per_launch": us, "bitwise_same_as_spmv": bool(torch.equal(ref, y)),
                     "max_rel_diff": float(((y - ref).abs() / ref.abs().clamp_min(1e-30)).max())}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
