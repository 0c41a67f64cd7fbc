"""Peaks measured once per box: pinned H2D / D2H bandwidth
(1 GiB, separately and concurrently), FP64 DFMA and FP32 FFMA throughput
(probe kernels in csrc/kernels_runtime.cu, 8 independent chains per thread,
4 CTAs of 256 per SM), L2 size, host cores.  Prints one JSON object.

    python tools/box_peaks.py > profiles/<round>_box_peaks.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2012_09646_b200 import dagrt as D
    dev = torch.cuda.current_device()
    prop = torch.cuda.get_device_properties(dev)
    out = {"gpu": prop.name, "sms": prop.multi_processor_count,
           "l2_bytes": getattr(prop, "L2_cache_size", None), "host_cores": os.cpu_count()}
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    out["h2d_gbs"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e6
    out["d2h_gbs"] = n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e6

    def both():
        ev = torch.cuda.Event()
        ev.record()
        for s, f in ((s1, lambda: d.copy_(h, non_blocking=True)), (s2, lambda: h2.copy_(d2, non_blocking=True))):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                f()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
    ms = timed(both)
    out["h2d_plus_d2h_concurrent_gbs"] = 2 * n / ms / 1e6

    ctx = D.Context(device=dev)
    buf = torch.zeros(1024, dtype=torch.float64, device="cuda")
    B = ctx.register_tensor("peak_out", buf)
    st = torch.cuda.Stream()
    grid, iters = 4 * prop.multi_processor_count, 1 << 16
    for name, key in (("peak_dfma", "fp64_fma_tflops"), ("peak_ffma", "fp32_fma_tflops")):
        L = ctx.prepare(name, grid, 256, [B, iters])
        L.raw(st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
            L.raw(st.cuda_stream)
            e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        fmas = grid * 256 * iters * 8
        out[key] = 2 * fmas / ms / 1e9
        out[key.replace("_tflops", "_ops_per_clk_per_sm_at_1965mhz")] = fmas / (ms * 1e-3) / (
            prop.multi_processor_count * 1.965e9)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
