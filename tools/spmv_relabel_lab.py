"""How much would a locality-preserving vertex order buy the HITS SpMVs?
Relabels the synthetic power-law graph by descending total degree (hubs
first, approximately undoing the generator's seeded random relabelling) and
times the HITS DAG (resident) and the product SpMV on both orders.  A lab
only: the product keeps the graph's own vertex ids.
    python tools/spmv_relabel_lab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def relabel(rp, ci, rpt, cit):
    import numpy as np
    n = rp.size - 1
    deg = np.diff(rp.astype(np.int64)) + np.diff(rpt.astype(np.int64))
    order = np.argsort(-deg, kind="stable")
    new = np.empty(n, np.int64)
    new[order] = np.arange(n)

    def perm(rp_, ci_):
        d = np.diff(rp_.astype(np.int64))
        rows = np.repeat(np.arange(n, dtype=np.int64), d)
        r2, c2 = new[rows], new[ci_.astype(np.int64)]
        key = r2 * n + c2
        idx = np.argsort(key, kind="stable")
        r2, c2 = r2[idx], c2[idx]
        rpn = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(r2, minlength=n), out=rpn[1:])
        return rpn.astype(np.int32), c2.astype(np.int32)
    a = perm(rp, ci)
    b = perm(rpt, cit)
    return a[0], a[1], b[0], b[1]


def main():
    import torch
    import synth
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200.programs import Hits
    g = synth.powerlaw_graph(synth.BASE_SEED, 20_000_000, 60_000_000, device="auto")
    out = {}
    for label, graph in (("generator_order", g), ("degree_order", relabel(*g))):
        ctx = D.Context(device=0)
        p = Hits(ctx, graph=graph)
        p.load_inputs(0)
        for _ in range(3):
            p.restart()
            p.run()
        ctx.sync()
        ms = []
        for _ in range(10):
            p.restart()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.run()
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        st = torch.cuda.Stream()
        L = p.it[0]
        for _ in range(3):
            L.raw(st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
            for _ in range(10):
                L.raw(st.cuda_stream)
            e1.record()
        e1.synchronize()
        out[label] = {"hits_dag_ms_median": ms[5], "spmv_us": e0.elapsed_time(e1) / 10 * 1e3}
        print(label, out[label], flush=True)
        del p
        ctx.close()
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
