"""Experiment: merge-path SpMV (spmv_merge) time vs the footprint of the gathered vector.

Same CSR structure as the HITS graph (BASELINE configs[4]); the column
indices are folded into the first N/f entries (ci % (N/f)) so that the
gathers touch an f-times smaller vector.  If the time drops with f, the
kernel is bound by L2 misses of the gathers, not by its streams.

    python tools/spmv_footprint.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import synth
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    from paper_2012_09646_b200.programs.hits_dl import spmv_out_bytes, spmv_plan
    n, e = 20_000_000, 60_000_000
    rp, ci, _, _ = synth.powerlaw_graph(synth.BASE_SEED, n, e)
    E = int(rp[-1])
    ob, grid = spmv_out_bytes(n, E)
    plan, pgrid, ws = spmv_plan(rp)
    ob = max(ob, 4 * n + ws)
    ctx = D.Context(device=0)
    t_rp = torch.from_numpy(rp).cuda()
    t_x = torch.rand(n, device="cuda")
    y = torch.zeros(ob // 4 + 1, device="cuda")
    A_rp = ctx.register_tensor("rp", t_rp)
    A_x = ctx.register_tensor("x", t_x)
    A_y = ctx.register_tensor("y", y)
    A_pl = ctx.register_tensor("plan", torch.from_numpy(plan).cuda())
    st = torch.cuda.Stream()
    out = {}
    for f in (1, 64):
        t_ci = torch.from_numpy((ci % (n // f)).astype(np.int32)).cuda()
        torch.cuda.synchronize()
        A_ci = ctx.register_tensor(f"ci{f}", t_ci)
        units = int(plan[0]) + -(-int(plan[1]) // 32) + int(plan[2])
        for kname in ("spmv_merge", "spmv_plan", "spmv_np"):
            if kname == "spmv_merge":
                L = ctx.prepare(kname, grid, 256, [A_rp, A_ci, A_x, A_y, n])
            elif kname == "spmv_np":  # same kernel, one CTA per unit (non-persistent)
                L = ctx.prepare("spmv_plan", units, 256, [A_rp, A_ci, A_pl, A_x, A_y, n])
            else:
                L = ctx.prepare(kname, pgrid, 256, [A_rp, A_ci, A_pl, A_x, A_y, n])
            for _ in range(3):
                L.raw(st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record()
                for _ in range(10):
                    L.raw(st.cuda_stream)
                e1.record()
            e1.synchronize()
            out[f"{kname}_fold{f}"] = e0.elapsed_time(e1) / 10 * 1e3
        ctx.unregister(A_ci)
        del t_ci
    # sorted-by-row gathers of a permuted-free vector: columns = row index (perfect locality)
    t_ci = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), np.diff(rp))).cuda()
    A_ci = ctx.register_tensor("cirow", t_ci)
    L = ctx.prepare("spmv_merge", grid, 256, [A_rp, A_ci, A_x, A_y, n])
    L.raw(st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record()
        for _ in range(10):
            L.raw(st.cuda_stream)
        e1.record()
    e1.synchronize()
    out["row_local"] = e0.elapsed_time(e1) / 10 * 1e3
    out["E"] = E
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
