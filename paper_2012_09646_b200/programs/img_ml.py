"""IMG and ML host programs (§V-B; Fig. 6; Fig. 10)."""
from __future__ import annotations

import os

import numpy as np
import torch

import synth
from .base import SMS, Program, grid_1d

# IMG readings R-IMG: (diameter, sigma^2); unsharp amount; extend factor
IMG_BLUR_S, IMG_BLUR_L, IMG_BLUR_U = (3, 0.1), (5, 10.0), (3, 5.0)
IMG_UNSHARP, IMG_EXTEND = 0.5, 5.0
IMG_COLS, IMG_THREADS = 512, 128  # stencil tile (csrc/kernels_img.cu)
IMG_ROWS = int(os.environ.get("DAGRT_IMG_ROWS", "64"))  # output rows per CTA (grid.y = ceil(h / rows))


class Images(Program):
    """Sharpen + low/medium-frequency blurs, combined by edge masks (4 streams)."""
    name = "img"

    def __init__(self, ctx, h=16384, w=16384, **kw):
        super().__init__(ctx, **kw)
        self.h, self.w = h, w
        n = h * w
        self.n = n
        stream = self.streaming
        self.alloc("img", n, torch.float32, mirror=stream)
        for name in ("bs", "bl", "bu", "ms", "ml", "iu", "i2"):
            self.alloc(name, n, torch.float32)
        self.alloc("i3", n, torch.float32, mirror=stream)
        self.alloc_red("mx")
        self.alloc_red("mn")
        self.inputs, self.sinks = ["img"], ["i3"]
        a = self.a
        sg = (max(1, -(-w // IMG_COLS)), max(1, -(-h // IMG_ROWS)))
        ge = grid_1d(n, 256, 4)
        gr = min(grid_1d(n, 256, 8), 1024)
        P = ctx.prepare
        self.L = [
            P("blur", sg, IMG_THREADS, [a["img"], a["bs"], h, w, IMG_BLUR_S[0], IMG_BLUR_S[1]]),
            P("blur", sg, IMG_THREADS, [a["img"], a["bl"], h, w, IMG_BLUR_L[0], IMG_BLUR_L[1]]),
            P("blur", sg, IMG_THREADS, [a["img"], a["bu"], h, w, IMG_BLUR_U[0], IMG_BLUR_U[1]]),
            P("sobel", sg, IMG_THREADS, [a["bs"], a["ms"], h, w]),
            P("sobel", sg, IMG_THREADS, [a["bl"], a["ml"], h, w]),
            P("maximum", gr, 256, [a["ml"], a["mx"], n]),
            P("minimum", gr, 256, [a["ml"], a["mn"], n]),
            P("extend", ge, 256, [a["ml"], a["mx"], a["mn"], n, IMG_EXTEND]),
            P("unsharpen", ge, 256, [a["img"], a["bu"], a["iu"], n, IMG_UNSHARP]),
            P("combine", ge, 256, [a["iu"], a["bl"], a["ml"], a["i2"], n]),
            P("combine", ge, 256, [a["i2"], a["bs"], a["ms"], a["i3"], n]),
        ]

    def _inputs(self, set_index=0):
        self.fill("img", synth.spec_img(self.h, self.w)["img"], set_index)

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        d0 = [io["img"]] if io else []
        L = self.L
        bs = g.kernel(L[0], d0)
        bl = g.kernel(L[1], d0)
        bu = g.kernel(L[2], d0)
        ms = g.kernel(L[3], [bs])
        ml = g.kernel(L[4], [bl])
        mx = g.kernel(L[5], [ml])
        mn = g.kernel(L[6], [ml])
        ex = g.kernel(L[7], [mx, mn])
        iu = g.kernel(L[8], [bu])
        i2 = g.kernel(L[9], [bl, ex, iu])
        i3 = g.kernel(L[10], [bs, ms, i2])
        self.graph_sinks(g, {"i3": i3})
        g.instantiate()
        return g

    def kernel_bytes(self):
        n = self.n * 4
        return {"blur_s": 2 * n, "blur_l": 2 * n, "blur_u": 2 * n, "sobel_s": 2 * n,
                "sobel_l": 2 * n, "maximum": n, "minimum": n, "extend": 2 * n,
                "unsharpen": 3 * n, "combine_1": 4 * n, "combine_2": 4 * n}


ML_C, ML_F = 10, 200  # classes (reading), features (L879-880)
NORM_THREADS = 512
MM_THREADS = 128  # csrc/kernels_ml.cu kMmThreads
NORM_GRID = 2 * SMS


def norm_smem(f):
    g_vec = f // 4 if f % 4 == 0 else f
    rl = max(NORM_THREADS // max(1, g_vec), NORM_THREADS // max(1, f), 1)
    return 8 * 3 * f * rl  # [row lanes][S, Qlo, Qhi] per column


def norm_stats_bytes(f, grid=None):
    """NORM `stats` array: header, fp64 mean/inv_sd, per-block S/Qlo/Qhi."""
    return 16 + 16 * f + 24 * f * (grid or NORM_GRID)


class MLEnsemble(Program):
    """Naive Bayes + Ridge Regression, softmax-normalised and averaged (L876-881)."""
    name = "ml"

    def __init__(self, ctx, n=10_000_000, f=ML_F, c=ML_C, **kw):
        super().__init__(ctx, **kw)
        self.n, self.f, self.c = n, f, c
        stream = self.streaming
        self.alloc("X", n * f, torch.int32, mirror=stream)
        self.alloc("Z", n * f, torch.float32)
        self.alloc("stats", 0, None, nbytes=norm_stats_bytes(f))
        for name, numel in (("theta", c * f), ("prior", c), ("W", c * f), ("b", c)):
            self.alloc(name, numel, torch.float32)
        for name in ("r1", "r2"):
            self.alloc(name, n * c, torch.float32)
        self.alloc("amax", n, torch.float32)
        self.alloc("l", n, torch.float32)
        self.alloc("r", n, torch.int32, mirror=stream)
        self.inputs, self.sinks = ["X"], ["r"]
        a = self.a
        P = ctx.prepare
        gr = grid_1d(n, 256, 2)
        # MMUL: 128 threads, persistent over 256-row tiles; W + padded X chunk in smem
        # MMUL (TMA path): 2 CTAs/SM, 64-row tiles double-buffered in smem
        gm = max(1, min(-(-n // (MM_THREADS // 2)), 2 * SMS))
        mm_smem = 4 * c * f + 16 + 2 * (MM_THREADS // 2) * 4 * f
        self.L = [
            P("norm", NORM_GRID, NORM_THREADS, [a["X"], a["Z"], a["stats"], n, f], smem=norm_smem(f)),
            P("nb_mmul", gm, MM_THREADS, [a["X"], a["theta"], a["prior"], a["r1"], n, f, c],
              smem=mm_smem),
            # rr_mmul (fp32 rows): 64 threads, two rows per thread (kernels_ml.cu
            # mmul_tma10<float, 2>: 1.36 vs 1.54 ms); nb_mmul keeps one row per
            # thread (its int->fp32 conversions run on the XU pipe: 2.34 vs 1.58 ms
            # with two rows per thread, tools/mmul_lab.py)
            P("rr_mmul", gm, MM_THREADS // 2, [a["Z"], a["W"], a["r2"], n, f, c], smem=mm_smem),
            P("rowmax", gr, 256, [a["r1"], a["amax"], n, c]),
            P("lse", gr, 256, [a["r1"], a["amax"], a["l"], n, c]),
            P("addv", gr, 256, [a["r2"], a["b"], n, c]),
            P("exp_sub", gr, 256, [a["r1"], a["l"], n, c]),
            P("softmax", gr, 256, [a["r2"], n, c]),
            P("softmax", gr, 256, [a["r1"], n, c]),
            P("argmax", gr, 256, [a["r1"], a["r2"], a["r"], n, c]),
        ]
        self.params = synth.ml_params(self.seed, f, c)
        for k, v in self.params.items():
            self.upload(k, v)

    def _inputs(self, set_index=0):
        self.fill("X", synth.spec_ml_x(self.n, self.f)["X"], set_index)

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        d0 = [io["X"]] if io else []
        L = self.L
        # NORM needs co-residency (software grid barrier): it is launched as a
        # kernel node like any other; the graph places it first on its branch.
        nrm = g.kernel(L[0], d0)
        nb = g.kernel(L[1], d0)
        rr = g.kernel(L[2], [nrm])
        mx = g.kernel(L[3], [nb])
        ls = g.kernel(L[4], [nb, mx])
        ad = g.kernel(L[5], [rr])
        ex = g.kernel(L[6], [mx, ls])
        s2 = g.kernel(L[7], [ad])
        s1 = g.kernel(L[8], [ex])
        am = g.kernel(L[9], [s2, s1])
        self.graph_sinks(g, {"r": am})
        g.instantiate()
        return g

    def kernel_bytes(self):
        n, f, c = self.n, self.f, self.c
        return {"norm": 12 * n * f, "nb_mmul": 4 * n * f + 4 * n * c, "rr_mmul": 4 * n * f + 4 * n * c,
                "rowmax": 4 * n * c + 4 * n, "lse": 4 * n * c + 8 * n, "addv": 8 * n * c,
                "exp_sub": 8 * n * c + 4 * n, "softmax_r2": 8 * n * c, "softmax_r1": 8 * n * c,
                "argmax": 8 * n * c + 4 * n}

    def f32(self, name):
        return self.t[name]
