"""VEC lab (BASELINE configs[0], N = 1M fp32, L2-resident): the product
square / reduce_diff at several grid sizes -- us per launch back to back on
one stream (CUDA events, 50 launches after 5) -- and the whole VEC DAG
(resident, 400 steps after 20) with the chosen grids swapped in.

    python tools/vec_lab.py [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    ctx = D.Context(device=0)
    p = bench.make_program("vec", ctx, "resident")
    p.load_inputs(0)
    p.run()
    ctx.sync()
    torch.cuda.synchronize()
    a, n = p.a, p.n
    st = torch.cuda.Stream()
    res = {}

    def b2b(L, reps=50):
        for _ in range(5):
            L.raw(st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
            for _ in range(reps):
                L.raw(st.cuda_stream)
            e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    for g in (148, 296, 489, 592, 1024, 2048):
        Ls = ctx.prepare("square", g, 256, [a["x"], a["x1"], n])
        Lr = ctx.prepare("reduce_diff", min(g, 1024), 256, [a["x1"], a["y1"], a["z"], n])
        r = {"square_us": round(b2b(Ls), 2), "reduce_diff_us": round(b2b(Lr), 2)}
        res[f"grid{g}"] = r
        print(g, json.dumps(r), flush=True)

    def dag_us(gs, gr, steps=400):
        p.L = [ctx.prepare("square", gs, 256, [a["x"], a["x1"], n]),
               ctx.prepare("square", gs, 256, [a["y"], a["y1"], n]),
               ctx.prepare("reduce_diff", gr, 256, [a["x1"], a["y1"], a["z"], n])]
        p._batch = p._steps = None
        ms = bench.time_steps(p.run, steps, 20, None)
        return ms / steps * 1e3

    for gs, gr in ((489, 489), (296, 296), (592, 592), (148, 148), (1024, 1024)):
        us = [round(dag_us(gs, gr), 2) for _ in range(3)]
        res[f"dag_sq{gs}_red{gr}"] = {"us_per_dag": us}
        print("dag", gs, gr, us, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
