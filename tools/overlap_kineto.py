"""Schedule evidence from HARDWARE timestamps: run one benchmark DAG under
torch.profiler (kineto -> CUPTI activity records: every kernel and memcpy the
process issues, including the scheduler's cuLaunchKernel launches, with the
GPU's own start/end times) and compute the paper's overlap metrics
(§V-F: CT, TC, CC, TOT) for the parallel scheduler and
the serial-sync baseline.  Unlike tools/overlap.py (events recorded on the
launch streams, whose start stamps complete when the stream reaches them,
not when the kernel gets SMs), these intervals are when the work ran.

    python tools/overlap_kineto.py --bench bs --mode stream --runs 2 --out gpurun_out/ov_bs_stream.json
(nsys is not in the image; the chrome trace written with --trace is the
timeline evidence.)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def device_intervals(trace):
    """[(kind, name, stream, start_ms, end_ms)] of GPU activity in a chrome trace."""
    out = []
    for ev in trace.get("traceEvents", []):
        cat = ev.get("cat", "")
        if cat not in ("kernel", "gpu_memcpy", "gpu_memset"):
            continue
        ts, dur = float(ev.get("ts", 0.0)), float(ev.get("dur", 0.0))
        kind = "kernel" if cat == "kernel" else ("memset" if cat == "gpu_memset" else "memcpy")
        name = ev.get("name", "")
        if kind == "memcpy":
            kind = "h2d" if "HtoD" in name else ("d2h" if "DtoH" in name else "d2d")
        out.append((kind, name, ev.get("args", {}).get("stream", -1), ts / 1e3, (ts + dur) / 1e3))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default="bs")
    ap.add_argument("--mode", default="stream")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--trace", default=None, help="write the parallel run's chrome trace here")
    args = ap.parse_args()
    import tempfile

    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200 import measure
    res = {"bench": args.bench, "mode": args.mode, "runs": args.runs,
           "source": "CUPTI activity records via torch.profiler (kineto)"}
    for policy in ("parallel", "serial"):
        ctx = D.Context(device=0, policy=policy)
        p = bench.make_program(args.bench, ctx, args.mode)
        p.load_inputs(0)
        for _ in range(2):
            p.restart()
            p.run()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(args.runs):
                p.restart()
                p.run()
            torch.cuda.synchronize()
        fd, path = tempfile.mkstemp(suffix=".json")
        os.close(fd)
        prof.export_chrome_trace(path)
        with open(path) as f:
            tr = json.load(f)
        os.unlink(path)
        iv = device_intervals(tr)
        # the HITS restart writes (host -> device) are input preparation, not DAG work
        K = [(a, b) for k, _, _, a, b in iv if k == "kernel"]
        T = [(a, b) for k, _, _, a, b in iv if k in ("h2d", "d2h")]
        m = measure.overlap(K, T)
        m["span_ms"] /= args.runs
        m["kernels"] = len(K) // args.runs
        m["transfers"] = len(T) // args.runs
        m["streams"] = len({s for k, _, s, _, _ in iv if k == "kernel"})
        res[policy] = m
        if policy == "parallel" and args.trace:
            keep = {"traceEvents": [e for e in tr.get("traceEvents", [])
                                    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]}
            with open(args.trace, "w") as f:
                json.dump(keep, f)
        ctx.close()
        del p
        torch.cuda.empty_cache()
    s = json.dumps(res)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
