"""f2 placement on one GPU (two slots backed by device 0): B&S DAG (10 x 10M
fp64 options, BASELINE configs[1]) resident on slot 0, through a Multi
context with data placement vs a plain context -- ms per DAG and the
placement decisions / migrations; and the stream form (inputs from pinned
host mirrors) where placement spreads the kernels.  On one physical GPU the
slots share SMs and HBM, so this measures the layer's overhead and its
decisions, not a multi-GPU speedup.
    python tools/multi_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import synth
    import synth.gpu as sg
    from paper_2012_09646_b200 import dagrt as D
    n, nv = 10_000_000, 10
    BS = (0.08, 0.30, 1.0, 60.0)
    sp = synth.spec_bs(n, nv)
    s = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nv)]
    for i in range(nv):
        sg.fill_tensor(s[i], synth.BASE_SEED, f"s{i}", sp[f"s{i}"])
    c = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nv)]
    torch.cuda.synchronize()
    out = {}
    one = torch.empty(1, dtype=torch.float64).pin_memory()

    def timed(run, steps=10, warm=3):
        for _ in range(warm):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            run()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / steps

    # plain context
    ctx = D.Context(device=0)
    S = [ctx.register_tensor(f"s{i}", s[i]) for i in range(nv)]
    Cc = [ctx.register_tensor(f"c{i}", c[i]) for i in range(nv)]
    Ls = [ctx.prepare("bs", 296, 256, [S[i], Cc[i], n, *BS]) for i in range(nv)]

    def run_ctx():
        for L in Ls:
            L()
        for i in range(nv):
            ctx.host_read(Cc[i], one.data_ptr(), 0, 8)
    out["single_context_ms"] = timed(run_ctx)
    ctx.close()
    # multi, data placement, inputs resident on slot 0
    for pol in ("data", "round_robin"):
        m = D.Multi(devices=[0, 0], placement=pol)
        MS = [m.register_tensor(f"s{i}", s[i], home=0) for i in range(nv)]
        MC = [m.register(f"c{i}", 8 * n) for i in range(nv)]
        placed = []

        def run_multi():
            placed.clear()
            for i in range(nv):
                placed.append(m.launch("bs", 296, 256, MS[i], MC[i], n, *BS))
            for i in range(nv):
                m.read(MC[i], one.data_ptr(), 0, 8)
            m.sync()
        out[f"multi_{pol}_resident_ms"] = timed(run_multi)
        out[f"multi_{pol}_placement"] = list(placed)
        out[f"multi_{pol}_stats"] = m.stats()
        m.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
