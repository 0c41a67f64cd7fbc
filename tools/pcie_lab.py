"""PCIe lab: pinned host -> device copy bandwidth of one large transfer on
one stream against the same bytes split over 2 / 4 streams, and D2H, and
H2D + D2H at once (stream mode is bound by these).

    python tools/pcie_lab.py
"""
import json


def main():
    import torch
    n = 1 << 28  # 1 GiB of fp32
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d2 = torch.empty(n, dtype=torch.float32, device="cuda")
    out = {}

    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            torch.cuda.synchronize()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    for k in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(k)]
        def h2d():
            part = n // k
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        ms = timed(h2d)
        out[f"h2d_{k}streams_GBps"] = round(4 * n / (ms * 1e-3) / 1e9, 1)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def d2h():
        with torch.cuda.stream(s1):
            h2.copy_(d2, non_blocking=True)
    ms = timed(d2h)
    out["d2h_GBps"] = round(4 * n / (ms * 1e-3) / 1e9, 1)
    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    ms = timed(both)
    out["h2d_plus_d2h_total_GBps"] = round(8 * n / (ms * 1e-3) / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
