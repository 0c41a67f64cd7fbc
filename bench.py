#!/usr/bin/env python
"""bench.py -- end-to-end ms per DAG of the run-time DAG scheduler (arXiv
2012.09646) on B200, next to its baselines, for the paper's six benchmarks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--bench vec|bs|img|ml|hits|dl|all]
                    [--impl dagrt|reference] [--no-cpu] [--no-baselines]

One step = one DAG of a benchmark through the whole hot path (SURVEY §8(a)
rows a1-a10): launches through the C ABI (dependency inference, stream
assignment, event wiring, prefetch), the sm_100a kernels, and the host
reads of the sinks.  By default ALL SIX benchmarks are measured (the suite,
BASELINE.json configs[0..4] at full size); the printed headline is B&S
(configs[1], 10 x 10M fp64 options) and the other five ride along under
"suite" (short DAGs -- VEC, the fp32 B&S -- over more steps, each
entry stating its own).  ``--bench X`` measures one benchmark only (its line
is the headline).

Printed JSON line (rank 0), headline benchmark:
  value      ms per DAG, job aggregate = max-over-ranks timed ms / DAGs done by
             all ranks; resident mode (inputs in HBM, host reads one element
             of each sink -- the Z[0] pattern of PAPER.md Fig. 4)
  e2e        the same through the C ABI with host buffers: inputs rewritten
             on the host before every step (untimed), H2D + D2H inside the
             timed region (first launch -> last host read returns, L819-820)
  baselines  serial-sync policy, the hand-written CUDA
             Graph with manual dependencies (L1062-1067), both modes; f1 graph
             cache, single-stream-children policy (L650-654), prefetch off
  dag_roofline  R_cp (slowest root->sink path's bytes at HBM bandwidth) and
             R_work (all bytes), as fractions of the measured time
  contention_free  Fig. 9 estimate (L1195-1201): serial per-vertex times
             summed along the DAG's longest path
  roofline   dominant kernel, event-timed live on its own launch stream while
             it runs alone (each launch of one DAG run repeated back to back on
             one stream) and inside the DAG; kernel_rooflines: every kernel
  cpu_baseline  the fp64 oracle on ONE pinned host core, bounded sample
Under torchrun each rank runs independent DAG instances on its own GPU (no
collective on the data path; NCCL only for the barrier and the max of the
timings) -> "scaling": "weak".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2012_09646_b200 import measure, replicas  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
ORDER = ["vec", "bs", "img", "ml", "hits", "dl", "bs_f32"]
HEADLINE = "bs"
PAPER_SIX = ("vec", "bs", "img", "ml", "hits", "dl")
UNIT = "ms per DAG"
METRIC = "end-to-end ms per DAG (resident inputs; job aggregate over GPUs)"

# Full BASELINE.json sizes per benchmark (configs[0..4])
FULL = {
    "vec": dict(n=1_000_000),
    "bs": dict(n=10_000_000),
    "img": dict(h=16384, w=16384),
    "ml": dict(n=10_000_000),
    "hits": dict(n=20_000_000, e=60_000_000),
    "dl": dict(h=16384, w=16384),
    "bs_f32": dict(n=10_000_000, dtype="f32"),  # the B&S DAG in fp32 (HBM-bound)
}
# the kernel whose roofline heads each line (the DAG's largest serial time share)
DOMINANT = {"vec": "square", "bs": "bs", "img": "blur", "ml": "norm", "hits": "spmv", "dl": "conv1",
            "bs_f32": "bs_f32"}
# device symbol of each dominant kernel (ncu names, profiles/*_traffic.json keys)
KSYM = {"square": "k_square", "bs": "k_bs2l_o6s3b2", "blur": "k_blur", "norm": "k_norm", "spmv": "k_spmv_split",
        "conv1": "k_conv1_r2b3", "conv2": "k_conv2_h", "bs_f32": "k_bs_f32"}
DTYPE = {"vec": "f32", "bs": "f64", "img": "f32", "ml": "f32/i32", "hits": "f32/i32", "dl": "f32", "bs_f32": "f32"}
WORKLOAD = {
    "vec": "VEC: 2 squares + sum of differences, N=1M fp32",
    "bs": "B&S: 10 independent Black-Scholes kernels, N=10M fp64 options each",
    "img": "IMG: blur/sobel/extend/unsharpen/combine, 16384x16384 fp32",
    "ml": "ML: Naive Bayes + Ridge Regression ensemble, 10M x 200",
    "hits": "HITS: 10 iterations CSR SpMV hub/authority, 20M-vertex power-law graph",
    "dl": "DL: two-branch CNN + dense merge, 2 x 16384x16384 fp32",
    "bs_f32": "B&S in fp32 (f4 variant): 10 independent kernels, N=10M fp32 options each",
}

SMS = 148
# DFMA + DMUL + DADD executed per option by the product B&S kernel (ncu
# dynamic instruction counts, profiles/) and the FP64 pipe's peak per SM per
# clock (ncu sm__sass_thread_inst_executed_op_dfma_pred_on.avg.peak_sustained;
# confirmed by the DFMA probe: 63.3 ops/clk/SM, profiles/r1_box_peaks.json).
BS_FP64_OPS_PER_OPTION = 37.5  # k_bs2l_o6s3b2: 39.5 DFMA+DMUL+DADD per option in ncu for the bs2t pricer, minus the two series terms the lean tables drop
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
    return PROGRAMS[name.split("_")[0]](ctx, mode=mode, share=share, **kw)


def time_steps(fn, steps, warmup, dist, prep=None):
    """Device time of `steps` calls of fn.  Without `prep`: one CUDA-event
    region around all steps (barrier + synchronize on both sides).  With
    `prep` (host-side input preparation before every step, e.g. HITS
    restarting from 1/sqrt(N)): each step is its own event-bracketed region
    (first launch -> the host holds the outputs) and the regions are summed;
    prep runs outside them."""
    import torch
    for _ in range(warmup):
        if prep:
            prep()
        fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if prep is None:
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
    else:
        ms = 0.0
        for _ in range(steps):
            prep()
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    if dist:
        ms = replicas.max_over_ranks(ms, dist, device="cuda")
        replicas.barrier(dist)
    return ms


def needs_prep(prog):
    """True if the program prepares its inputs on the host before a run (HITS)."""
    from paper_2012_09646_b200.programs.base import Program
    return type(prog).restart is not Program.restart or getattr(prog, "um", False)


def cpu_oracle_rate(name, budget_s=10.0):
    """Oracle (fp64, as it stands) on a bounded sample, on ONE host core:
    the process is pinned to one CPU (sched_setaffinity, like taskset) and
    BLAS pools are limited to one thread.  Returns (ms per DAG, sample
    text, cores)."""
    from threadpoolctl import threadpool_limits
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    try:
        if old:
            os.sched_setaffinity(0, {min(old)})
        with threadpool_limits(limits=1):
            return _cpu_oracle_rate(name, budget_s)
    finally:
        if old:
            os.sched_setaffinity(0, old)


def _cpu_oracle_rate(name, budget_s):
    import synth
    cores = 1
    if name in ("bs", "bs_f32"):
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


# ---------------------------------------------------------------- one benchmark
def fp64_floor_ms(n_options, mhz):
    return BS_FP64_OPS_PER_OPTION * n_options / (FP64_OPS_PER_SM_CLK * SMS * mhz * 1e6) * 1e3


def dag_of(D, name, prog, local, mode):
    """The inferred DAG of one run (a recording context on the same tensors)."""
    rctx = D.Context(device=local, record_dag=True)
    rp = make_program(name, rctx, mode, share=prog)
    rp.restart()
    rp.run()
    rctx.sync()
    verts, edges = rctx.dag()
    arr_index = {n: a.handle & 0xFFFFFFFF for n, a in rp.a.items()}
    rctx.close()
    return verts, edges, arr_index


def serial_vertex_times(D, name, prog, local, mode, runs=2):
    """Per-kernel (+ its H2D) and per-D2H times under serial scheduling (each
    kernel alone on the GPU), from the scheduler's event timeline."""
    sctx = D.Context(device=local, policy="serial")
    sp = make_program(name, sctx, mode, share=prog)
    sp.restart()
    sp.run()
    sctx.sync()
    acc_k, acc_h = None, {}
    for _ in range(runs):
        sp.restart()
        sctx.timeline(True)
        sp.run()
        items = sctx.timeline_export()
        sctx.timeline(False)
        vk = {}
        d2h = {}
        for kind, _s, vertex, ident, _b, t0, t1 in items:
            if kind in ("kernel", "h2d") and vertex >= 0:
                vk[vertex] = vk.get(vertex, 0.0) + (t1 - t0)
            elif kind == "d2h":
                d2h[ident] = d2h.get(ident, 0.0) + (t1 - t0)
        ks = [vk[v] for v in sorted(vk)]
        acc_k = ks if acc_k is None else [a + b for a, b in zip(acc_k, ks)]
        for k, v in d2h.items():
            acc_h[k] = acc_h.get(k, 0.0) + v
    sctx.close()
    return [x / runs for x in acc_k], {k: v / runs for k, v in acc_h.items()}


# Suite entries other than the headline: short DAGs are timed over more steps
# so that every timed region lasts a few milliseconds (VEC is ~0.03 ms per
# DAG: 10 steps would be a 0.3 ms region, dominated by the first step's
# host-side warm-up and event resolution).  The headline keeps EXACTLY
# --steps; each suite entry reports its own steps.
SUITE_STEP_SCALE = {"vec": 20, "bs_f32": 3}


def back_to_back_ms(prog, reps=5):
    """Each launch of one DAG run, alone on the GPU: repeated `reps` times back
    to back on one stream (raw launches of the same prepared arguments,
    through the C ABI) between CUDA events on that stream, so the interval is
    the kernels' execution (plus the ~1 us inter-kernel gaps) -- not the host
    launch latency a serial-sync region puts between an idle GPU's start
    event and the kernel.  Run after every DAG measurement of the program:
    in-place kernels (extend, exp_sub, addv, softmax) rewrite their arrays.
    Returns {kernel name: average ms per launch}."""
    import torch
    seq = prog.launch_sequence()
    st = torch.cuda.Stream()
    for L in seq:
        L.raw(st.cuda_stream)
    torch.cuda.synchronize()
    evs = []
    with torch.cuda.stream(st):
        for L in seq:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                L.raw(st.cuda_stream)
            e1.record()
            evs.append((L.kernel.name, e0, e1))
    torch.cuda.synchronize()
    acc = {}
    for kn, e0, e1 in evs:
        acc.setdefault(kn, []).append(e0.elapsed_time(e1) / reps)
    return {k: sum(v) / len(v) for k, v in acc.items()}


def bench_one(name, args, dist, local, world, peaks, full_report, steps=None):
    import torch
    from paper_2012_09646_b200 import dagrt as D
    K, W = (steps or args.steps), args.warmup
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    mhz = float(peaks.get("sm_max_mhz", 1965.0))

    # --- resident mode, parallel-async scheduler (the product)
    ctx = D.Context(device=local)
    prog = make_program(name, ctx, "resident")
    prog.load_inputs(0)
    dom = DOMINANT[name]
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
        t_end = time.perf_counter() + 0.3
        while time.perf_counter() < t_end:
            prog.run()
        torch.cuda.synchronize()
    per = ms / K
    value = replicas.job_ms_per_dag(ms, K, world)
    # dominant kernel inside the DAG: events on its own launch streams
    ctx.profile(dom, True)
    ms_prof = time_steps(prog.run, K, 0, dist)
    ctx.profile(dom, False)
    n_dag, sum_dag, busy_dag = ctx.profile_collect(dom)

    res = {}
    kb = prog.kernel_bytes()
    vbytes = list(kb.values())
    floor = None
    if name == "bs":
        floor = [fp64_floor_ms(prog.n, mhz)] * len(vbytes)
    verts, edges, arr_index = dag_of(D, name, prog, local, "resident")
    r_cp, r_work = measure.dag_rooflines(verts, edges, vbytes, peak, floor)

    # --- serial-sync baseline (+ the dominant kernel alone, event-timed)
    sctx = D.Context(device=local, policy="serial")
    sprog = make_program(name, sctx, "resident", share=prog)
    res["serial_resident_ms"] = time_steps(sprog.run, K, W, dist) / K
    # every kernel of the DAG alone on the GPU (serial policy), event-timed
    # per launch on its stream: the per-kernel roofline table
    knames = []
    for L in prog.launch_sequence():
        if L.kernel.name not in knames:
            knames.append(L.kernel.name)
    for kn in knames:
        sctx.profile(kn, True)
    time_steps(sprog.run, K, 0, dist)
    alone = {}
    for kn in knames:
        sctx.profile(kn, False)
        alone[kn] = sctx.profile_collect(kn)
    sctx.close()
    labels = list(kb.values())
    bytes_of = {}
    for L, nb in zip(prog.launch_sequence(), labels):
        bytes_of.setdefault(L.kernel.name, []).append(nb)
    kernel_rooflines = []
    for kn in knames:
        n_l, s_ms, _ = alone[kn]
        per_b = sum(bytes_of[kn]) / len(bytes_of[kn])
        avg = s_ms / max(1, n_l)
        ach = per_b / (avg * 1e-3) / 1e9 if avg > 0 else None
        kernel_rooflines.append({"kernel": kn, "launches_per_dag": len(bytes_of[kn]), "avg_launch_ms": avg,
                                 "algorithmic_bytes_per_launch": per_b, "achieved_gbs": ach,
                                 "hbm_frac": ach / peak if ach else None,
                                 "share_of_serial_dag": s_ms / max(1e-9, sum(a[1] for a in alone.values()))})
    kernel_rooflines.sort(key=lambda r: -r["share_of_serial_dag"])
    if dom not in alone:
        dom = kernel_rooflines[0]["kernel"]
    n_alone, sum_alone, busy_alone = alone[dom]
    if full_report:
        g = prog.graph()
        res["graph_resident_ms"] = time_steps(g.run, K, W, dist) / K
        del g
        for label, kw in (("f1_graph_cache", dict(graph_cache=True)),
                          ("single_stream", dict(policy="single_stream"))):
            c2 = D.Context(device=local, **kw)
            p2 = make_program(name, c2, "resident", share=prog)
            res[f"{label}_resident_ms"] = time_steps(p2.run, K, W, dist) / K
            if label == "f1_graph_cache":
                res["f1_graph_replays"] = c2.stats()["graph_replays"]
            c2.close()
        kms, _ = serial_vertex_times(D, name, prog, local, "resident")
        cf = measure.contention_free(verts, edges, kms)

    # --- end-to-end (stream mode) through the same C ABI with host buffers
    ectx = D.Context(device=local)
    eprog = make_program(name, ectx, "stream", share=prog)
    eprog.load_inputs(0)
    prep = eprog.restart if needs_prep(eprog) else None
    ectx.stats_reset()
    e2e_ms = time_steps(eprog.run, K, W, dist, prep)
    est = ectx.stats()
    steps_done = K + W
    h2d_ps = est["h2d_bytes"] / steps_done
    d2h_ps = est["d2h_bytes"] / steps_done
    if full_report:
        sectx = D.Context(device=local, policy="serial")
        seprog = make_program(name, sectx, "stream", share=eprog)
        res["serial_stream_ms"] = time_steps(seprog.run, K, W, dist, prep and seprog.restart) / K
        sectx.close()
        eg = eprog.graph()
        res["graph_stream_ms"] = time_steps(eg.run, K, W, dist, prep) / K
        del eg
        for label, kw in (("f1_graph_cache", dict(graph_cache=True)),
                          ("single_stream", dict(policy="single_stream")),
                          ("parallel_no_prefetch", dict(prefetch=False))):
            c2 = D.Context(device=local, **kw)
            p2 = make_program(name, c2, "stream", share=eprog)
            res[f"{label}_stream_ms"] = time_steps(p2.run, K, W, dist, prep and p2.restart) / K
            c2.close()
        # UM mode (§V-C): the stream workload on
        # managed arrays -- runtime prefetch vs GPU page faults, and the serial
        # page-fault baseline; pages go back to the host before every step
        # (restart(), outside the timed region)
        Ku = min(K, 5)
        for label, kw in (("um_parallel_prefetch", dict()), ("um_parallel_fault", dict(prefetch=False)),
                          ("um_serial_fault", dict(policy="serial", prefetch=False))):
            c2 = D.Context(device=local, **kw)
            p2 = make_program(name, c2, "um")
            p2.load_inputs(0)
            res[f"{label}_ms"] = time_steps(p2.run, Ku, W, dist, p2.restart) / Ku
            del p2
            c2.close()
            torch.cuda.empty_cache()
        # Fig. 9 in stream mode: serial kernel + H2D times, D2H on the host vertices
        sverts, sedges, s_arr = dag_of(D, name, eprog, local, "stream")
        skms, shms = serial_vertex_times(D, name, eprog, local, "stream")
        host_ms = {v[0]: shms.get(s_arr.get(v[2], -1), 0.0) for v in sverts if v[1] == "host"}
        cf_stream = measure.contention_free(sverts, sedges, skms, host_ms)
    e2e_per = e2e_ms / K

    # --- every kernel of the DAG alone, back to back on one stream (the
    # roofline's launch duration); the serial-sync event times stay beside it
    b2b = back_to_back_ms(prog)
    for kr in kernel_rooflines:
        kn = kr["kernel"]
        if kn in b2b:
            kr["avg_launch_ms_serial_sync"] = kr["avg_launch_ms"]
            kr["avg_launch_ms"] = b2b[kn]
            kr["achieved_gbs"] = kr["algorithmic_bytes_per_launch"] / (b2b[kn] * 1e-3) / 1e9
            kr["hbm_frac"] = kr["achieved_gbs"] / peak
            # repeated launches keep a working set below the 126 MB L2 warm:
            # those fractions are L2-assisted (VEC; the HITS l2norm's 80 MB)
            kr["l2_warm_back_to_back"] = kr["algorithmic_bytes_per_launch"] < 126e6
    sum_alone_serial = sum_alone
    if dom in b2b:
        sum_alone = b2b[dom] * n_alone

    # --- dominant-kernel roofline
    kpre = "bs" if dom == "bs_f32" else dom  # kernel_bytes() labels of the fp32 B&S are bs0..bs9
    per_launch = sum(v for k, v in kb.items() if k.startswith(kpre)) / max(1, sum(1 for k in kb if k.startswith(kpre)))
    avg_alone = sum_alone / max(1, n_alone)
    if name == "bs":
        # B&S is bound by whichever floor is higher: HBM (16 B/option) or the
        # FP64 pipe (BS_FP64_OPS_PER_OPTION ops/option); both are reported
        fpeak = FP64_OPS_PER_SM_CLK * SMS * mhz * 1e6 / 1e9
        ops = BS_FP64_OPS_PER_OPTION * prog.n / 1e9  # G fp64 ops per launch
        hbm_ach = per_launch / (avg_alone * 1e-3) / 1e9 if avg_alone > 0 else None
        fp64_ach = ops / (avg_alone * 1e-3) if avg_alone > 0 else None
        hbm_floor, fp64_floor = per_launch / (peak * 1e9), ops / fpeak
        fp64_info = {"pipe": "fp64", "fp64_achieved": fp64_ach, "fp64_peak": fpeak, "fp64_unit": "G fp64 ops/s",
                     "fp64_frac": fp64_ach / fpeak if fp64_ach else None,
                     "fp64_ops_per_option": BS_FP64_OPS_PER_OPTION,
                     "fp64_peak_source": f"{FP64_OPS_PER_SM_CLK} fp64 ops/clk/SM (ncu peak_sustained; DFMA probe "
                                         f"63.3) x {SMS} SMs x {mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"}
        if hbm_floor >= fp64_floor:
            roof = {"kernel": dom, "bound": "hbm", "achieved": hbm_ach, "peak": peak, "unit": "GB/s",
                    "frac": hbm_ach / peak if hbm_ach else None,
                    "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)", **fp64_info}
        else:
            roof = {"kernel": dom, "bound": "alu", "achieved": fp64_ach, "peak": fpeak, "unit": "G fp64 ops/s",
                    "frac": fp64_ach / fpeak if fp64_ach else None, **fp64_info,
                    "hbm_achieved_gbs": hbm_ach}
    else:
        ach = per_launch / (avg_alone * 1e-3) / 1e9 if avg_alone > 0 else None
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak if ach else None,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    roof.update({"traffic": None, "algorithmic_bytes_per_launch": per_launch, "launches": n_alone,
                 "avg_launch_ms": avg_alone,
                 "timing": "CUDA events on the kernel's stream around every launch of one DAG run, each "
                           "repeated 5x back to back (the kernel alone on the GPU, no host launch gaps)",
                 "avg_launch_ms_serial_sync": sum_alone_serial / max(1, n_alone),
                 "in_dag": {"launches": n_dag, "avg_launch_ms": sum_dag / max(1, n_dag), "busy_ms": busy_dag,
                            "union_achieved": (per_launch * n_dag / (busy_dag * 1e-3) / 1e9
                                               if name != "bs" and busy_dag > 0 else
                                               (BS_FP64_OPS_PER_OPTION * prog.n * n_dag / (busy_dag * 1e-3) / 1e9
                                                if busy_dag > 0 else None)),
                            "profiled_region_ms_per_step": ms_prof / K}})
    tr, tr_src = load_traffic(name, KSYM.get(dom, "k_" + dom))
    if tr is not None:
        roof["traffic"] = tr
        roof["traffic_source"] = tr_src

    out = {
        "value": value, "ms_per_step": per, "steps": K, "warmup": W, "dtype": DTYPE[name],
        "config": {"workload": WORKLOAD[name], "bench": name, "mode": "resident",
                   "l2": ("inputs larger than L2 (126 MB): no flush needed" if sum(vbytes) > 2 * 126e6
                          else "working set L2-resident at this size (BASELINE configs[0]); no flush"),
                   "parallelism": f"replicas x{world}"},
        "e2e": {"value": e2e_per / world, "unit": UNIT, "h2d_bytes_per_step": h2d_ps,
                "d2h_bytes_per_step": d2h_ps,
                "timed_region": "per step: first launch -> last host read returns; host input "
                                "preparation (restart) untimed" if prep else
                                "K steps back to back, inputs host-newer every step"},
        "gpu_launches": st["launches"],
        "roofline": roof,
        "kernel_rooflines": kernel_rooflines,
        "dag_roofline": {"R_cp_ms": r_cp, "R_work_ms": r_work, "frac_cp": r_cp / per,
                         "frac_work": r_work / per, "frac_bound": max(r_cp, r_work) / per,
                         "peak_gbs": peak,
                         "note": "R_cp = slowest root->sink path's algorithmic bytes at HBM bandwidth"
                                 + (" (B&S vertices: max of HBM and FP64-pipe time)" if name == "bs" else "")
                                 + "; R_work = all vertex bytes; frac = R / measured ms per DAG"},
        "clocks": clk.summary(),
        "scheduler": {"sched_us_per_launch": st["sched_ns"] / max(1, st["launches"]) / 1e3,
                      "breakdown_us_per_launch": {
                          k: st[f] / max(1, st["launches"]) / 1e3 for k, f in
                          (("cuLaunchKernel", "launch_ns"), ("cudaEventRecord", "record_ns"),
                           ("waits_and_h2d_enqueue", "wait_ns"))} | {
                          "bookkeeping": (st["sched_ns"] - st["launch_ns"] - st["record_ns"] - st["wait_ns"])
                          / max(1, st["launches"]) / 1e3},
                      "cross_stream_waits_per_dag": st["cross_stream_waits"] / K,
                      "streams": st["streams"]},
        "baselines": res,
        "speedup_vs_serial_resident": res["serial_resident_ms"] / per,
    }
    if full_report:
        out["vs_graph_resident"] = per / res["graph_resident_ms"]
        out["speedup_vs_serial_stream"] = res["serial_stream_ms"] / e2e_per
        out["vs_graph_stream"] = e2e_per / res["graph_stream_ms"]
        out["contention_free"] = {"resident_ms": cf, "stream_ms": cf_stream,
                                  "resident_frac": cf / per, "stream_frac": cf_stream / e2e_per,
                                  "method": "Fig. 9 (L1195-1201): per-vertex times under serial "
                                            "scheduling summed along the DAG's longest path"}
    for c in (ectx, ctx):
        c.close()
    del prog, eprog
    torch.cuda.empty_cache()
    return out


def geomean(xs):
    xs = [x for x in xs if x and x > 0]
    return math.exp(sum(math.log(x) for x in xs) / len(xs)) if xs else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--bench", default="all", choices=["all"] + ORDER)
    ap.add_argument("--impl", default="dagrt", choices=["dagrt", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-baselines", action="store_true", help="serial-sync baseline only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    # functional checks of the multi-rank path on a one-GPU box only (never a
    # measurement): DAGRT_BENCH_GPU pins every rank to one device and
    # DAGRT_DIST_BACKEND=gloo replaces NCCL (which refuses two ranks per GPU)
    if os.environ.get("DAGRT_BENCH_GPU") is not None:
        local = int(os.environ["DAGRT_BENCH_GPU"])
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        backend = os.environ.get("DAGRT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
        dist = tdist

    peaks, _ = load_peaks()
    names = ORDER if args.bench == "all" else [args.bench]
    head = HEADLINE if args.bench == "all" else args.bench
    results = {}
    for name in names:
        k = args.steps if name == head else args.steps * SUITE_STEP_SCALE.get(name, 1)
        results[name] = bench_one(name, args, dist, local, world, peaks, not args.no_baselines, k)

    if rank != 0:
        return
    h = results[head]
    cpu = None
    if world == 1 and not args.no_cpu:
        for name in names:
            v, sample, cores = cpu_oracle_rate(name)
            if v is not None:
                c = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                     "cpu_model": cpu_model(), "pinning": "sched_setaffinity to one core, BLAS 1 thread"}
                results[name]["cpu_baseline"] = c
                if name == head:
                    cpu = c
    out = {
        "metric": METRIC,
        "value": h["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": h["ms_per_step"],
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": h["dtype"],
        "data": "synthetic (seeded counter-based generator, synth/)",
        "config": h["config"],
        "e2e": h["e2e"],
        "gpu_launches": h["gpu_launches"],
        "roofline": h["roofline"],
        "dag_roofline": h["dag_roofline"],
        "cpu_baseline": cpu,
        "clocks": h["clocks"],
    }
    for k in ("scheduler", "baselines", "speedup_vs_serial_resident", "vs_graph_resident",
              "speedup_vs_serial_stream", "vs_graph_stream", "contention_free", "kernel_rooflines"):
        if k in h:
            out[k] = h[k]
    if len(names) > 1:
        out["suite"] = {n: {k: v for k, v in r.items() if k not in ("clocks",)} for n, r in results.items()
                        if n != head}
        # over the paper's six benchmarks (the fp32 B&S ablation variant is reported, not averaged in)
        six = [r for n, r in results.items() if n in PAPER_SIX]
        out["suite_geomean"] = {
            "over": [n for n in results if n in PAPER_SIX],
            "speedup_vs_serial_resident": geomean([r["speedup_vs_serial_resident"] for r in six]),
            "speedup_vs_serial_stream": geomean([r.get("speedup_vs_serial_stream") for r in six]),
            "vs_graph_resident": geomean([r.get("vs_graph_resident") for r in six]),
            "vs_graph_stream": geomean([r.get("vs_graph_stream") for r in six]),
            "dag_roofline_frac_cp": geomean([r["dag_roofline"]["frac_cp"] for r in six]),
            "dag_roofline_frac_work": geomean([r["dag_roofline"]["frac_work"] for r in six]),
        }
    print(json.dumps(out))


def run_reference(args, rank, world):
    """--impl reference: the oracle (as it stands) on ONE pinned host core, a
    bounded sample per step, same metric/unit/config as the dagrt arm's
    headline (B&S unless --bench names another)."""
    if rank != 0:
        return
    name = HEADLINE if args.bench == "all" else args.bench
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
    out = {"impl": "reference", "metric": METRIC,
           "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el / args.steps * 1e3, "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD[name], "bench": name},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "cpu_model": cpu_model(),
                            "sample": sample + f"; {budget}s per step, extrapolated to the full DAG"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
