"""SpMV hub-cache lab (BASELINE configs[4], the HITS graph in degree order):
the padded non-zero split with x[0, H) staged in shared memory
(csrc/spmv_common.cuh HUB; exp kernels spmv_hub4/2/1 = 256x4, 512x2,
1024x1 threads per SM) for several H, against the product "spmv".

For each configuration: us per launch of the two SpMVs of one HITS
iteration back to back on one stream (CUDA events, 10 pairs after 2), the
result compared bitwise with the product's; then the whole HITS DAG
(resident, 10 steps after 3) with both SpMV vertices swapped.

    python tools/spmv_hub_lab.py [--out FILE] [spec ...]
    spec = name:block:ctas_per_sm:hub_floats   e.g. spmv_hub1:1024:1:49152
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DEFAULT = ["spmv:256:4:0", "spmv_hub4:256:4:0", "spmv_hub4:256:4:8192", "spmv_hub4:256:4:12288",
           "spmv_hub2:512:2:16384", "spmv_hub2:512:2:24576", "spmv_hub1:1024:1:16384",
           "spmv_hub1:1024:1:32768", "spmv_hub1:1024:1:49152", "spmv_hub1:1024:1:56320"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-dag", action="store_true")
    ap.add_argument("specs", nargs="*")
    args = ap.parse_args()
    import torch
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()
    from paper_2012_09646_b200.programs import Hits
    ctx = D.Context(device=0)
    p = Hits(ctx)
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, n = p.a, p.n
    orig = list(p.it)
    warps_total = orig[0].grid.x * orig[0].block.x // 32  # the workspace holds this many warps
    st = torch.cuda.Stream()
    res, ref = {}, None
    for spec in (args.specs or DEFAULT):
        name, block, cps, hub = spec.split(":")
        block, cps, hub = int(block), int(cps), int(hub)
        grid = 148 * cps
        if grid * block // 32 > warps_total:
            grid = warps_total * 32 // block
        smem = 4 * hub
        argsets = [[a["rpt"], a["cit"], a["plant"], a["h1"], a["a2"], n],
                   [a["rp"], a["ci"], a["plan"], a["a1"], a["h2"], n]]
        Ls = [ctx.prepare(name, grid, block, A, smem) for A in argsets]
        p.it = orig  # the same x for every configuration (one product DAG from 1/sqrt(N)):
        p._batch = p._steps = None  # the DAG timings below move it
        p.restart()
        p.run()
        ctx.sync()
        torch.cuda.synchronize()
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
        y = torch.cat([p.vec("a2"), p.vec("h2")]).clone()
        if ref is None:
            ref = y
        r = {"grid": grid, "block": block, "hub_floats": hub, "us_per_launch": round(us, 2),
             "bitwise_same_as_product": bool(torch.equal(ref, y))}
        if not args.no_dag:
            it = list(orig)
            it[0], it[1] = Ls[0], Ls[1]
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
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                d0.record()
                p.run()
                d1.record()
                d1.synchronize()
                ms.append(d0.elapsed_time(d1))
            ctx.sync()
            ms.sort()
            r["hits_dag_ms_median"] = round(ms[len(ms) // 2], 4)
            p.it = orig
            p._batch = p._steps = None
        res[spec] = r
        print(spec, json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
