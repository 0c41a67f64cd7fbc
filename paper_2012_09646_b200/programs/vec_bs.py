"""VEC and Black & Scholes host programs (§V-B, Fig. 4, Fig. 6)."""
from __future__ import annotations

import os

import torch

import synth
from .base import Program, grid_1d

# B&S constants (readings R-BS in DESIGN.md; the paper prints none)
BS_R, BS_V, BS_T, BS_K = 0.08, 0.30, 1.0, 60.0


def bs_launch(name):
    """(block, dynamic shared memory) of a B&S pricing kernel: 256 threads,
    or for the warp-specialised bs3 forms (csrc/bs_math.cuh bs3_ws_body,
    named bs3_o<OPT>s<STAGES>b<CTAs/SM>) 8 consumer warps + 1 producer warp
    and a ring of STAGES chunks of 256 * OPT options in dynamic smem."""
    if name.startswith("bs3_"):
        opt, stages = int(name[5]), int(name[7])
        return 288, stages * 256 * opt * 8
    return 256, 0


# reduce_diff CTAs (deterministic last-block finish over this many partials)
VEC_RED_CTAS = int(os.environ.get("DAGRT_VEC_RED_CTAS", "1024"))


class Vec(Program):
    """x1 = x^2; y1 = y^2; z = sum(x1 - y1); host reads z[0] (Fig. 4)."""
    name = "vec"

    def __init__(self, ctx, n=1_000_000, **kw):
        super().__init__(ctx, **kw)
        self.n = n
        stream = self.streaming
        self.alloc("x", n, torch.float32, mirror=stream)
        self.alloc("y", n, torch.float32, mirror=stream)
        self.alloc("x1", n, torch.float32)
        self.alloc("y1", n, torch.float32)
        self.alloc_red("z")
        self.inputs, self.sinks = ["x", "y"], ["z"]
        a = self.a
        # one wave of 4 CTAs per SM (27.0 vs 28.1 us per VEC DAG with the
        # 489-CTA grid of 8 elements per thread, tools/vec_lab.py)
        g = grid_1d(n, 256, 4, waves=4)
        self.L = [
            ctx.prepare("square", g, 256, [a["x"], a["x1"], n]),
            ctx.prepare("square", g, 256, [a["y"], a["y1"], n]),
            ctx.prepare("reduce_diff", min(g, VEC_RED_CTAS), 256, [a["x1"], a["y1"], a["z"], n]),
        ]

    def _inputs(self, set_index=0):
        spec = synth.spec_vec(self.n)
        self.fill("x", spec["x"], set_index)
        self.fill("y", spec["y"], set_index)

    def result(self):
        return float(self.t["z"][:4].view(torch.float32)[0])

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        sx = g.kernel(self.L[0], deps=[io["x"]] if io else [])
        sy = g.kernel(self.L[1], deps=[io["y"]] if io else [])
        r = g.kernel(self.L[2], deps=[sx, sy])
        self.graph_sinks(g, {"z": r})
        g.instantiate()
        return g

    def kernel_bytes(self):
        n = self.n * 4
        return {"square_x": 2 * n, "square_y": 2 * n, "reduce_diff": 2 * n}


class BlackScholes(Program):
    """10 independent pricing kernels (L865-870); host reads each price vector."""
    name = "bs"

    def __init__(self, ctx, n=10_000_000, nvec=synth.BS_NVEC, dtype="f64", **kw):
        super().__init__(ctx, **kw)
        self.n, self.nvec, self.dtype = n, nvec, dtype
        stream = self.streaming
        tdt = torch.float64 if dtype == "f64" else torch.float32
        for i in range(nvec):
            self.alloc(f"s{i}", n, tdt, mirror=stream)
            self.alloc(f"c{i}", n, tdt, mirror=stream)
        self.inputs = [f"s{i}" for i in range(nvec)]
        self.sinks = [f"c{i}" for i in range(nvec)]
        if dtype == "f64":
            g = grid_1d(n, 256, 8, waves=2)  # one wave of the 2 resident CTAs/SM
            kname = "bs"
        else:  # f4: fp32 storage and arithmetic (HBM-bound)
            g = grid_1d(n, 256, 4, waves=8)
            kname = "bs_f32"
        self.L = [ctx.prepare(kname, g, 256, [self.a[f"s{i}"], self.a[f"c{i}"], n,
                                               BS_R, BS_V, BS_T, BS_K]) for i in range(nvec)]

    def _inputs(self, set_index=0):
        spec = synth.spec_bs(self.n, self.nvec)
        for i in range(self.nvec):
            if self.dtype == "f64":
                self.fill(f"s{i}", spec[f"s{i}"], set_index)
            elif not self.record:  # the same draws, rounded to fp32 (the oracle prices the rounded values)
                sp = (spec[f"s{i}"][0], spec[f"s{i}"][1], spec[f"s{i}"][2])
                tmp = torch.empty(self.n, dtype=torch.float64, device=self.device)
                import synth.gpu as sg
                sg.fill_tensor(tmp, self.seed + set_index, f"s{i}", sp)
                self.t[f"s{i}"].copy_(tmp)
                if f"s{i}" in self.mirror:
                    self.mirror[f"s{i}"].copy_(self.t[f"s{i}"])

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        for i, L in enumerate(self.L):
            k = g.kernel(L, deps=[io[f"s{i}"]] if io else [])
            self.graph_sinks(g, {f"c{i}": k}, only=[f"c{i}"])
        g.instantiate()
        return g

    def kernel_bytes(self):
        per = 16 if self.dtype == "f64" else 8
        return {f"bs{i}": per * self.n for i in range(self.nvec)}
