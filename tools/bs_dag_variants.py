"""B&S DAG (BASELINE configs[1], resident: 10 x 10M fp64, host reads one
element of each sink) with the pricing kernel swapped for each variant and
grid: ms per DAG (median of 10 after 3 warm-up, CUDA events around run()).
    python tools/bs_dag_variants.py [name:grid,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()
    from paper_2012_09646_b200.programs import BlackScholes
    from paper_2012_09646_b200.programs.vec_bs import BS_K, BS_R, BS_T, BS_V, bs_launch
    ctx = D.Context(device=0)
    p = BlackScholes(ctx)
    p.load_inputs(0)
    default = ["bs:296", "bs2l_o6s3b2:296", "bs2l_o4s3b3:444", "bs2t_o4s4b2:296", "bs2t_o4s3b3:444",
               "bs3_o6s4b2:296", "bs2t_o6s3b2:148", "bs:592", "bs2l_o6s3b2:296", "bs:296"]
    cases = sys.argv[1].split(",") if len(sys.argv) > 1 else default
    out = {}
    for case in cases:
        name, grid = case.split(":")
        block, smem = bs_launch(name)
        p.L = [ctx.prepare(name, int(grid), block, [p.a[f"s{i}"], p.a[f"c{i}"], p.n, BS_R, BS_V, BS_T, BS_K],
                           smem=smem) for i in range(p.nvec)]
        p._batch = p._steps = None
        for _ in range(3):
            p.run()
        ctx.sync()
        ms = []
        for _ in range(10):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.run()
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        key = case if case not in out else case + "_again"
        out[key] = {"ms_median": ms[5], "ms_min": ms[0]}
        print(case, round(ms[5], 4), flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
