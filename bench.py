#!/usr/bin/env python
"""bench.py -- end-to-end ms per DAG of the run-time DAG scheduler (arXiv
2012.09646) on B200, next to its baselines.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--bench bs|vec|img|ml|hits|dl]
                    [--impl dagrt|reference] [--suite]

One step = one DAG of the chosen benchmark through the whole hot path
(SURVEY §8(a) rows a1-a10): launches through the C ABI (dependency inference,
stream assignment, event wiring, prefetch), the sm_100a kernels, and the host
reads of the sinks.  The default workload is BASELINE.json configs[1]
(B&S, 10 x 10M fp64 options).

Printed JSON line (rank 0):
  value      ms per DAG, job aggregate = max-over-ranks timed ms / DAGs done by
             all ranks; resident mode (inputs in HBM, host reads one element
             of each sink -- the Z[0] pattern of PAPER.md Fig. 4)
  e2e        the same through the C ABI with host buffers: inputs rewritten
             on the host every step, H2D + D2H inside the timed region
  baselines  serial-sync policy and the hand-written
             CUDA Graph with manual dependencies (L1062-1067), both modes
  roofline   dominant kernel, timed live with events on its launch stream
  cpu_baseline  the fp64 oracle on this host on a bounded sample (rank 0, N=1)
Under torchrun each rank runs independent DAG instances on its own GPU (no
collective on the data path; NCCL only for the barrier and the max of the
timings) -> "scaling": "weak".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2012_09646_b200 import replicas  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

# Full BASELINE.json sizes per benchmark (configs[0..4])
FULL = {
    "vec": dict(n=1_000_000),
    "bs": dict(n=10_000_000),
    "img": dict(h=16384, w=16384),
    "ml": dict(n=10_000_000),
    "hits": dict(n=20_000_000, e=60_000_000),
    "dl": dict(h=16384, w=16384),
}
DOMINANT = {"vec": "square", "bs": "bs", "img": "blur", "ml": "norm", "hits": "spmv", "dl": "conv1"}
# device symbol of each dominant kernel (ncu names, profiles/*_traffic.json keys)
KSYM = {"square": "k_square", "bs": "k_bs_l3b2", "blur": "k_blur", "norm": "k_norm", "spmv": "k_spmv",
        "conv1": "k_conv1_r2b3"}
DTYPE = {"vec": "f32", "bs": "f64", "img": "f32", "ml": "f32/i32", "hits": "f32/i32", "dl": "f32"}
WORKLOAD = {
    "vec": "VEC: 2 squares + sum of differences, N=1M fp32",
    "bs": "B&S: 10 independent Black-Scholes kernels, N=10M fp64 options each",
    "img": "IMG: blur/sobel/extend/unsharpen/combine, 16384x16384 fp32",
    "ml": "ML: Naive Bayes + Ridge Regression ensemble, 10M x 200",
    "hits": "HITS: 10 iterations CSR SpMV hub/authority, 20M-vertex power-law graph",
    "dl": "DL: two-branch CNN + dense merge, 2 x 16384x16384 fp32",
}


SMS = 148
# DFMA + DMUL + DADD executed per option by k_bs (ncu dynamic instruction
# counts, profiles/r1_summary.md) and the FP64 pipe's peak per SM per clock
# (ncu sm__sass_thread_inst_executed_op_dfma_pred_on.avg.peak_sustained).
BS_FP64_OPS_PER_OPTION = 46  # 46.4 measured (gpurun_out fp64_bs2.csv -> profiles/)
FP64_OPS_PER_SM_CLK = 64


def load_traffic(bench, kernel):
    """DRAM bytes per launch of `kernel` from the newest committed ncu summary
    (profiles/<round>_traffic.json, written by tools/collect_profiles.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    for p in reversed(files):
        try:
            with open(p) as f:
                v = json.load(f).get(bench, {}).get(kernel)
        except (OSError, ValueError):
            continue
        if v is not None:
            return v, os.path.relpath(p, ROOT)
    return None, None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def make_program(name, ctx, mode, share=None, size=None):
    from paper_2012_09646_b200.programs import PROGRAMS
    kw = dict(FULL[name] if size is None else size)
    kw.pop("e", None) if name != "hits" else None
    return PROGRAMS[name](ctx, mode=mode, share=share, **kw)


def time_steps(fn, steps, warmup, dist):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        ms = replicas.max_over_ranks(ms, dist, device="cuda")
        replicas.barrier(dist)
    return ms


def cpu_oracle_rate(name, budget_s=10.0):
    """Oracle (fp64, as it stands) on a bounded sample; returns (ms per DAG,
    sample text, cores).  BLAS thread pools are limited to one thread so the
    core count is exact."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        return _cpu_oracle_rate(name, budget_s)


def _cpu_oracle_rate(name, budget_s):
    import numpy as np
    import synth
    cores = 1  # numpy is single-threaded here (BLAS pools limited above)
    if name == "bs":
        from oracle import bs as obs
        n = FULL["bs"]["n"]
        chunk = 1_000_000
        spec = synth.spec_bs(chunk)["s0"]
        s = synth.draw(synth.BASE_SEED, "s0", spec)
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s and done < 10 * n:
            obs.call(s)
            done += chunk
        el = time.perf_counter() - t0
        return el / done * 10 * n * 1e3, f"{done} of {10 * n} options (1M-option chunks)", cores
    if name == "vec":
        from oracle import vec as ov
        n = FULL["vec"]["n"]
        spec = synth.spec_vec(n)
        x = synth.draw(synth.BASE_SEED, "x", spec["x"])
        y = synth.draw(synth.BASE_SEED, "y", spec["y"])
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s and reps < 200:
            ov.vec(x, y)
            reps += 1
        el = time.perf_counter() - t0
        return el / reps * 1e3, f"{reps} full DAGs", cores
    # The other four: the whole oracle DAG on a strip (IMG, DL: full-width
    # row bands; ML: a row block) or a smaller graph of the same recipe
    # (HITS), repeated within the budget and extrapolated linearly in the
    # work unit (pixels, rows, vertices + edges) to one full-size DAG.
    if name == "img":
        from oracle import img as oi
        rows, w = 128, FULL["img"]["w"]
        im = synth.draw(synth.BASE_SEED, "img", synth.spec_img(rows, w)["img"]).reshape(rows, w)
        fn = lambda: oi.img_pipeline(im)  # noqa: E731
        scale, sample = FULL["img"]["h"] / rows, f"{rows}x{w} row band"
    elif name == "ml":
        from oracle import ml as om
        rows, f = 20_000, 200
        X = synth.draw(synth.BASE_SEED, "X", synth.spec_ml_x(rows, f)["X"]).reshape(rows, f)
        p = synth.ml_params(synth.BASE_SEED, f, 10)
        fn = lambda: om.ml(X, p["theta"], p["prior"], p["W"], p["b"])  # noqa: E731
        scale, sample = FULL["ml"]["n"] / rows, f"{rows}x{f} row block"
    elif name == "hits":
        from oracle import hits as oh
        n, e = 200_000, 600_000
        g = synth.powerlaw_graph(synth.BASE_SEED, n, e)
        fn = lambda: oh.hits(*g)  # noqa: E731
        full = FULL["hits"]["n"] + FULL["hits"]["e"]
        scale, sample = full / (n + len(g[1])), f"{n}-vertex {len(g[1])}-edge graph, same recipe, 10 iterations"
    elif name == "dl":
        from oracle import dl as odl
        rows, w = 64, FULL["dl"]["w"]
        sp = synth.spec_dl(rows, w)
        x = synth.draw(synth.BASE_SEED, "x", sp["x"]).reshape(rows, w)
        y = synth.draw(synth.BASE_SEED, "y", sp["y"]).reshape(rows, w)
        w1, w2, wd = (synth.draw(synth.BASE_SEED, k, sp[k]) for k in ("w1", "w2", "wd"))
        fn = lambda: odl.dl(x, y, w1, w2, wd)  # noqa: E731
        scale, sample = FULL["dl"]["h"] / rows, f"two {rows}x{w} row bands"
    else:
        return None, "not implemented", cores
    reps, t0 = 0, time.perf_counter()
    while reps == 0 or time.perf_counter() - t0 < budget_s:
        fn()
        reps += 1
    el = time.perf_counter() - t0
    return el / reps * scale * 1e3, f"{reps} x oracle DAG on a {sample}, x{scale:.0f} to one DAG", cores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--bench", default="bs", choices=list(FULL))
    ap.add_argument("--impl", default="dagrt", choices=["dagrt", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-baselines", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    from paper_2012_09646_b200 import dagrt as D
    name = args.bench
    K, W = args.steps, args.warmup

    # --- resident mode, parallel-async scheduler (the product)
    ctx = D.Context(device=local)
    prog = make_program(name, ctx, "resident")
    prog.load_inputs(0)
    dom = DOMINANT[name]
    ctx.profile(dom, False)
    # nvidia-smi samples every 100 ms and takes ~0.2 s to start: the sampler
    # runs from before the warm-up through the timed region (same load), so
    # short regions (B&S: ~5 ms) still get clock samples
    with Clocks(local) as clk:
        time.sleep(0.3)
        for _ in range(W):
            prog.run()
        torch.cuda.synchronize()
        ctx.stats_reset()
        ms = time_steps(prog.run, K, 0, dist)
        st = ctx.stats()  # launches etc. of exactly the K timed steps
        # keep the GPU under the same load until the sampler has seen it
        t_end = time.perf_counter() + 0.3
        while time.perf_counter() < t_end:
            prog.run()
        torch.cuda.synchronize()
    value = replicas.job_ms_per_dag(ms, K, world)
    # roofline: the same K steps again with the dominant kernel's launches
    # bracketed by CUDA events on their own launch streams (kept out of the
    # `value` region: the events add host work the baselines do not pay)
    ctx.profile(dom, True)
    ms_prof = time_steps(prog.run, K, 0, dist)
    ctx.profile(dom, False)
    n_launch, sum_ms, busy_ms = ctx.profile_collect(dom)

    # --- baselines and end-to-end (stream) mode
    res = {}
    if not args.no_baselines:
        sctx = D.Context(device=local, policy="serial")
        sprog = make_program(name, sctx, "resident", share=prog)
        res["serial_resident_ms"] = time_steps(sprog.run, K, W, dist) / K
        g = prog.graph()
        res["graph_resident_ms"] = time_steps(g.run, K, W, dist) / K
    ectx = D.Context(device=local)
    eprog = make_program(name, ectx, "stream", share=prog)
    eprog.load_inputs(0)
    ectx.stats_reset()
    e2e_ms = time_steps(eprog.run, K, W, dist)
    est = ectx.stats()
    steps_done = K + W
    h2d_ps = est["h2d_bytes"] / steps_done
    d2h_ps = est["d2h_bytes"] / steps_done
    if not args.no_baselines:
        sectx = D.Context(device=local, policy="serial")
        seprog = make_program(name, sectx, "stream", share=eprog)
        res["serial_stream_ms"] = time_steps(seprog.run, K, W, dist) / K
        eg = eprog.graph()
        res["graph_stream_ms"] = time_steps(eg.run, K, W, dist) / K
        # NEXT(f1): the same scheduler with deferred submission + batch graph cache
        cctx = D.Context(device=local, graph_cache=True)
        cprog = make_program(name, cctx, "resident", share=prog)
        res["f1_graph_cache_resident_ms"] = time_steps(cprog.run, K, W, dist) / K
        res["f1_graph_replays"] = cctx.stats()["graph_replays"]
        csctx = D.Context(device=local, graph_cache=True)
        csprog = make_program(name, csctx, "stream", share=eprog)
        res["f1_graph_cache_stream_ms"] = time_steps(csprog.run, K, W, dist) / K
        # ablation: the parallel scheduler with the
        # prefetcher off -- each H2D is issued on its consumer's own stream
        # (L356-366 / L662-664 describe the prefetch this removes)
        nctx = D.Context(device=local, prefetch=False)
        nprog = make_program(name, nctx, "stream", share=eprog)
        res["parallel_no_prefetch_stream_ms"] = time_steps(nprog.run, K, W, dist) / K

    if rank != 0:
        return
    peaks, peak_src = load_peaks()
    kb = prog.kernel_bytes()
    dom_bytes = sum(v for k, v in kb.items() if k.startswith(dom))
    per_launch = dom_bytes / max(1, sum(1 for k in kb if k.startswith(dom)))
    achieved = (per_launch * n_launch) / (busy_ms * 1e-3) / 1e9 if busy_ms > 0 else None
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None, "traffic": None,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": per_launch,
            "launches": n_launch, "avg_launch_ms": sum_ms / max(1, n_launch), "busy_ms": busy_ms,
            "profiled_region_ms_per_step": ms_prof / K,
            "note": "achieved = algorithmic bytes of all timed launches / union of their "
                    "event-timed intervals on their launch streams, over a second K-step "
                    "region run right after the value region"}
    total_bytes = sum(kb.values())
    roof["dag_work_roofline_ms"] = total_bytes / (peak * 1e9) * 1e3
    if name == "bs" and busy_ms > 0:
        # B&S is bound by the FP64 pipe, not HBM: report against it
        n_opt = FULL["bs"]["n"]
        ops = BS_FP64_OPS_PER_OPTION * n_opt * n_launch / (busy_ms * 1e-3) / 1e9
        mhz = float(peaks.get("sm_max_mhz", 1965.0))
        fpeak = FP64_OPS_PER_SM_CLK * SMS * mhz * 1e6 / 1e9
        roof.update({"bound": "alu", "pipe": "fp64", "achieved": ops, "peak": fpeak,
                     "unit": "G fp64 ops/s", "frac": ops / fpeak,
                     "peak_source": f"{FP64_OPS_PER_SM_CLK} fp64 ops/clk/SM (ncu peak_sustained) x "
                                    f"{SMS} SMs x {mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                     "fp64_ops_per_option": BS_FP64_OPS_PER_OPTION,
                     "hbm_achieved_gbs": achieved, "hbm_frac": achieved / peak if achieved else None})
    tr, tr_src = load_traffic(name, KSYM[dom])
    if tr is not None:
        roof["traffic"] = tr
        roof["traffic_source"] = tr_src
    cpu = None
    if world == 1 and not args.no_cpu:
        v, sample, cores = cpu_oracle_rate(name)
        if v is not None:
            cpu = {"value": v, "unit": "ms per DAG", "cores": cores, "kind": "oracle",
                   "sample": sample}
    out = {
        "metric": "end-to-end ms per DAG (resident inputs; job aggregate over GPUs)",
        "value": value,
        "unit": "ms",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms / K,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE[name],
        "data": "synthetic (seeded counter-based generator, synth/)",
        "config": {"workload": WORKLOAD[name], "bench": name, "mode": "resident",
                   "l2": "inputs larger than L2 (126 MB)" if total_bytes > 2 * 126e6
                   else "working set L2-resident; no flush", "parallelism": f"replicas x{world}"},
        "e2e": {"value": e2e_ms / K / world, "unit": "ms per DAG", "h2d_bytes_per_step": h2d_ps,
                "d2h_bytes_per_step": d2h_ps},
        "gpu_launches": st["launches"],
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "scheduler": {"sched_us_per_launch": st["sched_ns"] / max(1, st["launches"]) / 1e3,
                      "cross_stream_waits_per_dag": st["cross_stream_waits"] / K,
                      "streams": st["streams"]},
    }
    if res:
        out["baselines"] = res
        per = ms / K
        out["speedup_vs_serial_resident"] = res["serial_resident_ms"] / per
        out["vs_graph_resident"] = per / res["graph_resident_ms"]
        out["speedup_vs_serial_stream"] = res["serial_stream_ms"] / (e2e_ms / K)
        out["vs_graph_stream"] = (e2e_ms / K) / res["graph_stream_ms"]
    print(json.dumps(out))


def run_reference(args, rank, world):
    """--impl reference: the oracle (as it stands) on this host's cores, a
    bounded sample per step, same metric/unit/config as the dagrt arm."""
    if rank != 0:
        return
    name = args.bench
    budget = 2.0
    vals = []
    for _ in range(args.warmup):
        cpu_oracle_rate(name, budget_s=0.2)
    t0 = time.perf_counter()
    sample = ""
    for _ in range(args.steps):
        v, sample, cores = cpu_oracle_rate(name, budget_s=budget)
        vals.append(v)
    el = time.perf_counter() - t0
    v = statistics.median(vals) if vals and vals[0] is not None else None
    out = {"impl": "reference", "metric": "end-to-end ms per DAG (resident inputs; job aggregate over GPUs)",
           "value": v, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el / args.steps * 1e3, "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD[name], "bench": name},
           "cpu_baseline": {"value": v, "unit": "ms per DAG", "cores": 1, "kind": "oracle",
                            "sample": sample + f"; {budget}s per step, extrapolated to the full DAG"},
           "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
