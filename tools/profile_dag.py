"""Run one benchmark DAG a few times (for ncu capture).

    python tools/profile_dag.py --bench ml [--runs 2] [--scale 1.0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default="bs")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--mode", default="resident")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2012_09646_b200 import dagrt as D
    ctx = D.Context(device=0)
    p = bench.make_program(args.bench, ctx, args.mode)
    p.load_inputs(0)
    for _ in range(args.runs):
        p.run()
    ctx.sync()
    torch.cuda.synchronize()
    print("done", args.bench)


if __name__ == "__main__":
    main()
