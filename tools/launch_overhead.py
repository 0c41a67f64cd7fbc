"""Host-side cost of the scheduler per launch (C++ time from dagrt_stats and
Python-inclusive wall time), against raw launches and a CUDA graph.

    python tools/launch_overhead.py [--n 2000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    args = ap.parse_args()
    import torch
    from paper_2012_09646_b200 import dagrt as D
    out = {}
    ctx = D.Context(device=0)
    a = torch.zeros(1024, device="cuda")
    b = torch.zeros(1024, device="cuda")
    torch.cuda.synchronize()
    A = ctx.register_tensor("a", a)
    B = ctx.register_tensor("b", b)
    chain = ctx.prepare("square", 1, 256, [A, B, 1024])     # a -> b
    back = ctx.prepare("square", 1, 256, [B, A, 1024])      # b -> a (dependent chain)
    indep = [ctx.prepare("square", 1, 256, [A, ctx.register_tensor(f"o{i}", torch.zeros(1024, device="cuda")), 1024])
             for i in range(8)]
    torch.cuda.synchronize()
    for name, seq in (("dependent_chain", [chain, back]), ("fan_out_8", indep)):
        for _ in range(3):
            for L in seq:
                L()
        ctx.sync()
        ctx.stats_reset()
        t0 = time.perf_counter()
        k = 0
        while k < args.n:
            for L in seq:
                L()
                k += 1
        t1 = time.perf_counter()
        ctx.sync()
        t2 = time.perf_counter()
        st = ctx.stats()
        out[name] = {"host_us_per_launch_incl_python": (t1 - t0) / k * 1e6,
                     "sched_us_per_launch_cxx": st["sched_ns"] / k / 1e3,
                     "gpu_drain_ms": (t2 - t1) * 1e3,
                     "cross_stream_waits": st["cross_stream_waits"] / k}
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    t0 = time.perf_counter()
    for _ in range(args.n):
        chain.raw(sp)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out["raw_launch_us_incl_python"] = (t1 - t0) / args.n * 1e6
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
