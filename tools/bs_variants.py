"""Time the B&S kernel tuning variants (same math) on one 10M-option vector."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import synth
    import synth.gpu as sg
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    n = 10_000_000
    ctx = D.Context(device=0)
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, dtype=torch.float64, device="cuda")
    sg.fill_tensor(s, 20120964, "s0", synth.spec_bs(n)["s0"])
    S = ctx.register_tensor("s", s)
    Cc = ctx.register_tensor("c", c)
    st = torch.cuda.Stream()
    out = {}
    ref = None
    sel = sys.argv[1].split(",") if len(sys.argv) > 1 else None
    for name, waves in (("bs", 2), ("bs_p1b6", 6), ("bs_p2b3", 3), ("bs_p2b4", 4), ("bs_p4b2", 2),
                        ("bs_a3b4", 4), ("bs_a5b4", 4), ("bs_a7b4", 4), ("bs_a5b3", 3),
                        ("bs_l4b2", 2), ("bs_l2b3", 3), ("bs_l2b4", 4), ("bs_l1b4", 4),
                        ("bs_l3b2", 2), ("bs_l3b3", 3), ("bs_l8b1", 1),
                        ("bs2_p3w2b2", 2), ("bs2_p2w2b3", 3), ("bs2_p2w4b2", 2), ("bs2_p4w2b2", 2),
                        ("bs2_p1w2b4", 4), ("bs2t_o4s4b2", 2), ("bs2t_o4s3b3", 3), ("bs2t_o2s4b4", 4),
                        ("bs2t_o6s3b2", 2), ("bs3_o6s4b2", 2), ("bs3_o6s6b2", 2), ("bs3_o4s8b2", 2),
                        ("bs3_o4s6b3", 3), ("bs3_o2s8b4", 4), ("bs2l_o6s3b2", 2), ("bs2l_o4s3b3", 3),
                        ("bs2l_o6s3b3", 3), ("bs2l_o6s2b3", 3), ("bs2l_o8s2b2", 2),
                        ("bs2m_o6s3b2", 2), ("bs2m_o4s3b3", 3), ("bs2m_o6s3b3", 3), ("bs2m_o8s2b2", 2),
                        ("bs2m_o4s4b2", 2), ("bs2c_o6s3b2", 2), ("bs2x_o6s3b2", 2),
                        ("bs3_o6s4b2l", 2), ("bs3_o6s6b2l", 2), ("bs3_o4s6b3l", 3), ("bs3_o4s8b2l", 2)):
        if sel and name not in sel:
            continue
        from paper_2012_09646_b200.programs.vec_bs import bs_launch
        block, smem = bs_launch(name)
        for grid_mult in (1, 2, 4):
            grid = 148 * waves * grid_mult
            L = ctx.prepare(name, grid, block, [S, Cc, n, 0.08, 0.30, 1.0, 60.0], smem=smem)
            for _ in range(3):
                L.raw(st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record()
                for _ in range(20):
                    L.raw(st.cuda_stream)
                e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            if ref is None:
                ref = c.clone()
            same = bool(torch.equal(ref, c))
            rel = float(((ref - c).abs() / (ref.abs() + 1e-12)).max())
            out[f"{name}_g{grid}"] = {"us": us, "GBps": 16 * n / us / 1e3, "bitwise_same": same, "max_rel_vs_first": rel}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
