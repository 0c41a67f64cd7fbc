"""f1 (graph cache) lab: ms per DAG of each benchmark, resident, for the
eager scheduler, the hand-written CUDA graph, the graph cache with one
event-record node per vertex (DAGRT_F1_EVENTS=vertex), with none (vertex
events stand for their stream's tail in the graph: tail) and with nodes only
for the records the eager first issue saw escape (the default: learn).
Each arm is timed twice, interleaved (CUDA events, K steps after W).

    python tools/f1_lab.py [--benches vec,bs,...] [--steps K] [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--benches", default="vec,bs,img,ml,hits,dl")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    out = {}
    for name in a.benches.split(","):
        ctx = D.Context(device=0)
        prog = bench.make_program(name, ctx, "resident")
        prog.load_inputs(0)
        arms = {}

        def t(label, fn, p):
            prep = p.restart if bench.needs_prep(p) else None
            k = {"vec": 25, "bs": 5}.get(name, 1) * a.steps  # >= ~3 ms per timed region
            ms = bench.time_steps(fn, k, a.warmup, None, prep) / k
            arms.setdefault(label, []).append(round(ms, 5))

        g = prog.graph()
        for _ in range(a.reps):
            t("eager", prog.run, prog)
            t("hand_graph", g.run, prog)
            for label, env in (("f1_vertex_events", "vertex"), ("f1_tail_only", "tail"), ("f1_learn", "learn")):
                os.environ["DAGRT_F1_EVENTS"] = env
                c2 = D.Context(device=0, graph_cache=True)
                p2 = bench.make_program(name, c2, "resident", share=prog)
                t(label, p2.run, p2)
                c2.close()
        del g
        os.environ.pop("DAGRT_F1_EVENTS", None)
        ctx.close()
        torch.cuda.empty_cache()
        out[name] = {k: sorted(v)[len(v) // 2] for k, v in arms.items()}  # median
        out[name]["runs"] = arms
        print(name, json.dumps(out[name]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
