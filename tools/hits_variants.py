"""HITS DAG (BASELINE configs[4], resident) with the SpMV vertices swapped
for experimental kernels: ms per DAG (10 steps after 3 warm-up, CUDA events),
and the a1 result compared with the product's.
    python tools/hits_variants.py [name,name,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()
    from paper_2012_09646_b200.programs import Hits
    ctx = D.Context(device=0)
    p = Hits(ctx)
    p.load_inputs(0)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["spmv", "spmv_pad_l2", "spmv_pad2", "spmv"]
    orig = list(p.it)
    out, ref = {}, None
    for name in names:
        it = list(orig)
        for i in (0, 1):
            L = orig[i]
            it[i] = ctx.prepare(name, L.grid.x, L.block.x, [p.a[k] for k in (("rpt", "cit", "plant", "h1", "a2") if i == 0
                                                                                  else ("rp", "ci", "plan", "a1", "h2"))]
                                + [p.n])
        p.it = it
        p._batch = p._steps = None
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
        ctx.sync()
        a1 = p.t["a1"].clone()
        if ref is None:
            ref = a1
        ms.sort()
        out[name + ("" if name not in out else "_again")] = {
            "ms_per_dag_median": ms[len(ms) // 2], "ms_min": ms[0],
            "max_rel_diff_a1": float(((a1 - ref).abs() / ref.abs().clamp_min(1e-30)).max())}
        print(name, round(ms[len(ms) // 2], 3), flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
