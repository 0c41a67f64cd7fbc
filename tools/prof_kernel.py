"""Launch one benchmark kernel (a few times) at its full BASELINE size, for
ncu captures:  ncu --set full -k regex:k_spmv_nz -c 1 -o out python tools/prof_kernel.py spmv
    python tools/prof_kernel.py spmv|bs|conv2 [kernel names...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import synth
    import synth.gpu as sg
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    what = sys.argv[1]
    names = sys.argv[2:]
    ctx = D.Context(device=0)
    st = torch.cuda.Stream()
    if what == "spmv":
        from paper_2012_09646_b200.programs.hits_dl import spmv_nz_grid, spmv_out_bytes, spmv_pad_plan
        n, e = 20_000_000, 60_000_000
        rp, ci, _, _ = synth.powerlaw_graph(synth.BASE_SEED, n, e, device="auto")
        E = int(rp[-1])
        ob, grid = spmv_out_bytes(n, E)
        g = spmv_nz_grid(E + n)
        ob = max(ob, 4 * n + 16 + 12 * 8 * g)
        t = {"rp": torch.from_numpy(rp).cuda(), "ci": torch.from_numpy(ci).cuda(),
             "plan": torch.from_numpy(spmv_pad_plan(rp, ci)).cuda(), "x": torch.rand(n, device="cuda"),
             "y": torch.zeros(ob // 4 + 1, device="cuda")}
        torch.cuda.synchronize()
        A = {k: ctx.register_tensor(k, v) for k, v in t.items()}
        Ls = {"spmv": ctx.prepare("spmv", g, 256, [A["rp"], A["ci"], A["plan"], A["x"], A["y"], n]),
              "spmv_merge": ctx.prepare("spmv_merge", grid, 256, [A["rp"], A["ci"], A["x"], A["y"], n])}
    elif what == "bs":
        n = 10_000_000
        s = torch.empty(n, dtype=torch.float64, device="cuda")
        c = torch.empty(n, dtype=torch.float64, device="cuda")
        sg.fill_tensor(s, synth.BASE_SEED, "s0", synth.spec_bs(n)["s0"])
        S, Cc = ctx.register_tensor("s", s), ctx.register_tensor("c", c)
        Ls = {k: ctx.prepare(k, 296 if "b2" in k or k == "bs" else 444, 256, [S, Cc, n, 0.08, 0.30, 1.0, 60.0])
              for k in (names or ["bs"])}
        names = []
    elif what == "conv2":
        from paper_2012_09646_b200.programs import DeepLearning
        p = DeepLearning(ctx, h=16384, w=16384)
        p.load_inputs(0)
        p.run()
        ctx.sync()
        from paper_2012_09646_b200.programs.hits_dl import CONV2_ROWS_CFG, CONV2_WS_CFG, conv2_ws_launch
        a = p.a
        (_, _), (h2, w2), _ = p.shapes
        Ls = {"conv2": p.L[4]}
        for v in list(CONV2_WS_CFG) + list(CONV2_ROWS_CFG):
            th, sm = conv2_ws_launch(v)
            Ls[v] = ctx.prepare(v, 148, th, [a["px"], a["w2"], a["c2x"], h2, w2], smem=sm)
    else:
        raise SystemExit(f"unknown {what}")
    for k in (names or list(Ls)):
        for _ in range(3):
            Ls[k].raw(st.cuda_stream)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
