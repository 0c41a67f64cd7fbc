"""HITS L2-norm lab (BASELINE configs[4]: 20M fp32): the product l2norm
against the cp.async.bulk-ring variants (exp l2norm_t<NST>x<KB>) for several
grids; us per launch back to back (CUDA events, 20 after 2), HBM fraction of
the algorithmic 4 B/element, the result compared with the product's.

    python tools/l2norm_lab.py [--out FILE]
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
    D.load_experimental()
    peak = float(bench.load_peaks()[0].get("hbm_gbs", 6548.0))
    n = 20_000_000
    ctx = D.Context(device=0)
    v = torch.rand(n, device="cuda")
    out = torch.zeros(8 + 8 * 1024, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    V = ctx.register_tensor("v", v)
    O = ctx.register_tensor("o", out)
    st = torch.cuda.Stream()
    res, ref = {}, None
    confs = [("l2norm", 592), ("l2norm_r2", 1024), ("l2norm_t2x16", 296), ("l2norm_t3x12", 296),
             ("l2norm_t4x8", 592)]
    src = torch.rand(n, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
    for name, grid in confs:
        L = ctx.prepare(name, grid, 256, [V, O, n])
        r = {"grid": grid}
        # three L2 states: warm (the same vector back to back), producer-written
        # (v rewritten just before, as the HITS DAG's SpMV output is), cold
        # (a 256 MB buffer written in between)
        for state in ("warm", "written", "cold"):
            ts = []
            for it in range(12):
                if state == "written":
                    v.copy_(src)
                elif state == "cold":
                    flush.fill_(float(it))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(400000)  # the GPU is busy while the host enqueues: no launch latency inside
                e0.record()
                L.raw(torch.cuda.current_stream().cuda_stream)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts = sorted(ts[2:])
            r[f"us_{state}"] = round(ts[len(ts) // 2], 2)
        r0 = float(out[:4].view(torch.float32)[0])
        if ref is None:
            ref = r0
        r["rel_diff_vs_first"] = abs(r0 - ref) / ref
        res[f"{name}_g{grid}"] = r
        print(name, json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
