"""HITS and DL host programs (§V-B; Fig. 6)."""
from __future__ import annotations

import math
import os

import torch

import synth
from .base import SMS, Program, grid_1d

CONV2_TC_SMEM = 2 * 9 * 512 + 2 * 9 * 4096 + 64    # csrc/kernels_conv_tc.cu kTcSmem (conv2_tc1/tc2/tc3)
CONV2_TC_THREADS = 128
# conv2_tma<MODE> dynamic shared memory (csrc/kernels_conv_tc.cu tma_smem<MODE>):
# 1 KB alignment slack + 3 x 36 KB TMA stages + lo (and hi) A tiles + B tiles + barriers
CONV2_TMA_SMEM = {m: 1024 + 3 * 9 * 4096 + (2 if m == 0 else 1) * 9 * 4096 + 2 * 9 * 512 + 64 for m in (0, 1, 2)}
# two-group TMA kernels (conv2_tmag<MODE>, 256 threads): 1 (MODE 0) / 2 stages per group, A tiles per group
CONV2_TMAG_SMEM = {m: 1024 + 2 * (1 if m == 0 else 2) * 9 * 4096 + 2 * (2 if m == 0 else 1) * 9 * 4096
                   + 2 * 9 * 512 + 64 for m in (0, 1)}
# input-row ring TMA kernel (conv2_tmar, 288 threads): 12 slots x 12 KB + 2 groups' lo tiles + B + barriers
CONV2_TMAR_SMEM = 1024 + 12 * 3 * 4096 + 2 * 9 * 4096 + 2 * 9 * 512 + 256
CONV2_TMAR_THREADS = 288
# product "conv2" = conv2_tman3x1 (TMA-gathered A, three consumer groups with one
# TMA stage each, 3xTF32 in two MMA chains); csrc/kernels_conv_tc.cu tmang_smem<3, 1>
CONV2_TMAN_THREADS = 384  # round-1 product, now the variant "conv2_tman3x1"
CONV2_TMAN_SMEM = 1024 + 3 * 9 * 4096 + 3 * 9 * 4096 + 2 * 9 * 512 + 64
G2TC = 2 * 148                                    # persistent tcgen05 CTAs (2 per SM)
# warp-specialised conv2 (csrc/kernels_conv2.cu c2ws::Cfg<S, NB, SW>): S TMA
# stages, NB TMEM buffers, SW split warps -> (threads, dynamic shared memory)
CONV2_WS_CFG = {"conv2_ws": (4, 2, 4), "conv2_ws6": (6, 2, 4), "conv2_ws6s8": (6, 2, 8),
                "conv2_ws6b3": (6, 3, 4), "conv2_ws5s8b3": (5, 3, 8)}
# row-staged conv2 (c2rows::Cfg<R, NB, SW>): R input-row slots of 8704 B
CONV2_ROWS_CFG = {"conv2_rows": (12, 2, 8), "conv2_rows_s4": (12, 2, 4), "conv2_rows_r20": (20, 2, 8)}
# one-MMA-per-tap fp16-split conv2 (c2h::Cfg<R, NB, SW>): B is 9 x 1 KB as in c2ws
CONV2_H_CFG = {"conv2_h": (12, 3, 4), "conv2_h_s8": (12, 3, 8), "conv2_h_b4": (16, 4, 4), "conv2_h_s12": (12, 3, 12),
               "conv2_h_s8b2": (12, 2, 8), "conv2_h_s8r16": (16, 3, 8), "conv2_h_s16": (12, 3, 16),
               "conv2_h_s24": (12, 3, 24), "conv2_h_s12b4": (12, 4, 12), "conv2_h_s24b4": (12, 4, 24),
               "conv2_h_r16": (16, 3, 12), "conv2_h_r20": (20, 3, 12), "conv2_h_r24": (24, 3, 12)}


CONV2_HS_CFG = {"conv2_hs": (8, 3, 12), "conv2_hs_r12": (12, 3, 12), "conv2_hs_s8": (8, 3, 8),
                "conv2_hs_s16": (8, 3, 16)}


def conv2_ws_launch(name):
    if name in CONV2_HS_CFG:  # A in shared memory: + NB x 9 taps x 4 KB
        r, nb, sw = CONV2_HS_CFG[name]
        return 32 * (6 + sw), 1024 + r * 8704 + 9 * 1024 + nb * 9 * 4096 + 8 * (2 * r + 3 * nb) + 16
    if name in CONV2_ROWS_CFG or name in CONV2_H_CFG:
        r, nb, sw = CONV2_ROWS_CFG.get(name) or CONV2_H_CFG[name]
        return 32 * (6 + sw), 1024 + r * 8704 + 9 * 1024 + 8 * (2 * r + 3 * nb) + 16
    s, nb, sw = CONV2_WS_CFG[name]
    return 32 * (6 + sw), 1024 + s * 9 * 4096 + 9 * 1024 + 8 * (2 * s + 3 * nb) + 16


CONV2_WS_THREADS, CONV2_WS_SMEM = conv2_ws_launch("conv2_ws")
# product "conv2" = k_conv2_h<12, 3, 12> (csrc/kernels_conv2.cu): 148 persistent CTAs
CONV2_H_CFG["conv2"] = (12, 3, 12)
CONV2_GRID = 148
CONV2_THREADS, CONV2_SMEM = conv2_ws_launch("conv2")
CONV2_TC5_SMEM = 2 * 9 * 512 + 3 * 3 * 4 * 129 * 16 + 2 * 2 * 9 * 4096 + 64  # kC3Smem (conv2_tc5, 384 thr, 148 CTAs)
HITS_ITERS = 10          # reading; parity unpinned (constant)
SPMV_TILE = 32 * 8       # merge items per warp tile (csrc/kernels_hits.cu)
SPMV_WARPS = 8           # warps per 256-thread CTA


# Row classes of the planned SpMV (csrc/kernels_hits.cu k_spmv_plan; the
# kernel traps if a plan was built with other bounds).
SPMV_SHORT_MAX = 4        # deg <= 4: thread per row
SPMV_LONG_MIN = 256       # deg > 256: chunks of SPMV_LONG_CHUNK non-zeros, CTA per chunk
SPMV_LONG_CHUNK = 2048
SPMV_MED_ROWS_PER_CTA = 32
SPMV_CTAS = 148 * 8       # persistent grid
SPMV_SHORT_ROWS_PER_CTA = 1024
SPMV_PLAN_HEADER = 16


def spmv_plan(row_ptr):
    """Row-class plan of a CSR for k_spmv_plan, built once when the graph is
    registered (the graph is static and resident).

    Layout (int32): header[16] = (NL, NM, NS, short_max, long_min, chunk, 0..),
    NL long chunks as (row, k_begin, first chunk of the row, chunks of the
    row), then the NM medium row ids.  Returns (plan, grid, workspace bytes
    needed after y's N floats)."""
    import numpy as np
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.size - 1
    deg = np.diff(rp)
    long_rows = np.nonzero(deg > SPMV_LONG_MIN)[0]
    med = np.nonzero((deg > SPMV_SHORT_MAX) & (deg <= SPMV_LONG_MIN))[0].astype(np.int32)
    nch = (deg[long_rows] + SPMV_LONG_CHUNK - 1) // SPMV_LONG_CHUNK
    nl = int(nch.sum())
    items = np.zeros((nl, 4), dtype=np.int64)
    if nl:
        first = np.repeat(np.cumsum(nch) - nch, nch)              # first chunk of each chunk's row
        rows = np.repeat(long_rows, nch)
        within = np.arange(nl) - first
        items[:, 0] = rows
        items[:, 1] = rp[rows] + within * SPMV_LONG_CHUNK
        items[:, 2] = first
        items[:, 3] = np.repeat(nch, nch)
    ns = -(-n // SPMV_SHORT_ROWS_PER_CTA)
    header = np.zeros(SPMV_PLAN_HEADER, dtype=np.int64)
    header[:6] = (nl, med.size, ns, SPMV_SHORT_MAX, SPMV_LONG_MIN, SPMV_LONG_CHUNK)
    plan = np.concatenate([header, items.ravel(), med.astype(np.int64)]).astype(np.int32)
    units = nl + -(-med.size // SPMV_MED_ROWS_PER_CTA) + ns
    return plan, max(1, min(units, SPMV_CTAS)), 16 + 8 * nl


# merge-path SpMV grid: 8 CTAs per SM = two waves of the 4 that fit (64
# registers x 256 threads); shorter per-warp merge ranges balance the two
# concurrent SpMVs of a HITS iteration better: HITS DAG 8.16 ms vs 8.30 with
# one persistent wave (2: 10.8, 3: 9.8, 12: 8.20, 16: 8.21 ms)
SPMV_CTAS_PER_SM = int(os.environ.get("DAGRT_SPMV_CTAS_PER_SM", "8"))


# non-zero-split SpMV ("spmv" = csrc/kernels_hits.cu k_spmv_nz)
NZ_CHUNK = 128
NZ_MAGIC = 0x4E5A3031
NZ_HEADER = 16
NZ_CTAS_PER_SM = int(os.environ.get("DAGRT_SPMV_NZ_CTAS_PER_SM", "8"))  # two waves of 4 resident (<= 64 registers): 251 vs 257 us (tools/spmv_lab.py)


def spmv_nz_plan(row_ptr):
    """Row structure of a CSR re-encoded for k_spmv_nz, built once when the
    graph is registered (the graph is static and resident):
    int32 [header(16) | rbase(nc + 1) | flags(ceil(E/32) + 4 words) | nzrow(nr)]
      flags: bit k set iff non-zero k is the first of its (non-empty) row;
      nzrow: ids of the non-empty rows in order;
      rbase[c]: ordinal (index into nzrow) of the row holding non-zero c*128.
    Returns the plan array."""
    import numpy as np
    rp = np.asarray(row_ptr, dtype=np.int64)
    e = int(rp[-1])
    deg = np.diff(rp)
    ne = deg > 0
    nzrow = np.nonzero(ne)[0].astype(np.int64)
    starts = rp[:-1][ne]
    nwords = (e + 31) // 32 + 4
    # distinct powers of two per word: their sum is their OR (exact in fp64)
    flags = np.bincount(starts >> 5, weights=np.left_shift(1, starts & 31).astype(np.float64),
                        minlength=nwords).astype(np.uint64).astype(np.uint32)
    nc = (e + NZ_CHUNK - 1) // NZ_CHUNK
    rbase = np.searchsorted(starts, np.arange(nc + 1, dtype=np.int64) * NZ_CHUNK, side="right") - 1
    rbase = np.maximum(rbase, 0)
    off_r = NZ_HEADER
    off_f = off_r + nc + 1
    off_f += (-off_f) % 4  # 16-byte aligned flag words
    off_n = off_f + nwords
    plan = np.zeros(off_n + max(1, nzrow.size), dtype=np.int32)
    plan[:8] = (NZ_MAGIC, nc, nzrow.size, NZ_CHUNK, off_r, off_f, off_n, e)
    plan[off_r:off_r + nc + 1] = rbase
    plan[off_f:off_f + nwords] = flags.view(np.int32)
    plan[off_n:off_n + nzrow.size] = nzrow
    return plan


PAD_MAGIC = 0x50414430


def spmv_pad_plan(row_ptr, col_idx):
    """The CSR re-encoded for the product SpMV (k_spmv_pad), once, when the
    graph is registered: every empty row gets one column index -1 (value 0),
    so row ordinals are row ids.
    int32 [header(16) | rp2(N+1) | rbase(nc+1) | flags(4nc+4) | ci2(E2)]:
      rp2   padded row pointers, E2 = rp2[N] = E + #empty rows;
      flags bit k set iff item k starts its row (every row starts one item);
      rbase[c] row holding item c*128;  ci2 the padded column indices, the
            last chunk filled up with -1 (whole 128-item chunks)."""
    import numpy as np
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int64)
    n = rp.size - 1
    deg = np.diff(rp)
    pdeg = np.maximum(deg, 1)
    rp2 = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(pdeg, out=rp2[1:])
    e2 = int(rp2[-1])
    # whole chunks (the tail padded with -1) so that chunk copies stay in bounds
    ci2 = np.full(max(-(-e2 // NZ_CHUNK) * NZ_CHUNK, 1), -1, dtype=np.int64)
    if ci.size:
        row_of = np.repeat(np.arange(n, dtype=np.int64), deg)
        ci2[rp2[row_of] + (np.arange(ci.size, dtype=np.int64) - rp[row_of])] = ci
    starts = rp2[:-1]
    nc = (e2 + NZ_CHUNK - 1) // NZ_CHUNK
    nwords = 4 * nc + 4
    flags = np.bincount(starts >> 5, weights=np.left_shift(1, starts & 31).astype(np.float64),
                        minlength=nwords).astype(np.uint64).astype(np.uint32)
    rbase = np.searchsorted(starts, np.arange(nc + 1, dtype=np.int64) * NZ_CHUNK, side="right") - 1
    rbase = np.maximum(rbase, 0)
    off_rp = NZ_HEADER
    off_rb = off_rp + n + 1
    off_f = off_rb + nc + 1
    off_f += (-off_f) % 4
    off_c = off_f + nwords
    off_c += (-off_c) % 4
    plan = np.zeros(off_c + ci2.size, dtype=np.int32)
    plan[:9] = (PAD_MAGIC, nc, n, NZ_CHUNK, off_rp, off_rb, off_f, off_c, e2)
    plan[off_rp:off_rp + n + 1] = rp2
    plan[off_rb:off_rb + nc + 1] = rbase
    plan[off_f:off_f + nwords] = flags.view(np.int32)
    plan[off_c:off_c + ci2.size] = ci2
    return plan


def spmv_nz_grid(e):
    nc = -(-e // NZ_CHUNK)
    return max(1, min(-(-nc // SPMV_WARPS), NZ_CTAS_PER_SM * SMS))


def spmv_out_bytes(n, e):
    """(bytes of an SpMV output: N floats + 3 workspace words per warp, grid)."""
    ntiles = -(-(n + e) // SPMV_TILE)
    grid = max(1, min(-(-ntiles // SPMV_WARPS), SPMV_CTAS_PER_SM * SMS))
    return 4 * n + 16 + 12 * SPMV_WARPS * grid, grid


def degree_order(graph, device="auto"):
    """The graph relabelled by descending total degree (hubs first): returns
    (row_ptr, col_idx, row_ptr_t, col_idx_t) of P A P^T and new_id (old vertex
    id -> new id).  Rows keep sorted columns.  A registration-time re-encoding
    like the SpMV plans (outside the timed region): the DAG is unchanged, the
    hub and authority vectors live in the new order (the scores of vertex v
    are at new_id[v]).  On the HITS graph the gathers of the SpMVs then hit a
    compact hot region of x: SpMV 218 vs 252 us, HITS DAG 4.90 vs 5.78 ms
    (tools/spmv_relabel_lab.py)."""
    import numpy as np
    rp, ci, rpt, cit = graph
    n = rp.size - 1
    use_torch = False
    if device == "auto":
        try:
            use_torch = torch.cuda.is_available()
        except Exception:
            use_torch = False
    if use_torch:
        dev = torch.device("cuda")
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.int64)).to(dev)  # noqa: E731
        drp, drpt = torch.diff(t(rp)), torch.diff(t(rpt))
        order = torch.sort(-(drp + drpt), stable=True).indices
        new = torch.empty(n, dtype=torch.int64, device=dev)
        new[order] = torch.arange(n, device=dev)

        def perm(rp_, ci_):
            d = torch.diff(t(rp_))
            rows = torch.repeat_interleave(torch.arange(n, device=dev), d)
            key = new[rows] * n + new[t(ci_)]
            key = torch.sort(key).values
            r2, c2 = key // n, key % n
            rpn = torch.zeros(n + 1, dtype=torch.int64, device=dev)
            rpn[1:] = torch.cumsum(torch.bincount(r2, minlength=n), 0)
            return rpn.to(torch.int32).cpu().numpy(), c2.to(torch.int32).cpu().numpy()
        a, b = perm(rp, ci), perm(rpt, cit)
        return (a[0], a[1], b[0], b[1]), new.cpu().numpy()
    deg = np.diff(rp.astype(np.int64)) + np.diff(rpt.astype(np.int64))
    order = np.argsort(-deg, kind="stable")
    new = np.empty(n, np.int64)
    new[order] = np.arange(n)

    def perm_np(rp_, ci_):
        d = np.diff(rp_.astype(np.int64))
        rows = np.repeat(np.arange(n, dtype=np.int64), d)
        key = np.sort(new[rows] * n + new[ci_.astype(np.int64)])
        r2, c2 = key // n, key % n
        rpn = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(r2, minlength=n), out=rpn[1:])
        return rpn.astype(np.int32), c2.astype(np.int32)
    a, b = perm_np(rp, ci), perm_np(rpt, cit)
    return (a[0], a[1], b[0], b[1]), new


class Hits(Program):
    """HITS hub/authority iteration with two SpMV branches per iteration (L882-886).

    ``vertex_order``: "degree" (default) registers the graph relabelled by
    descending degree (degree_order(); ``self.new_id`` maps the given ids to
    the registered ones, ``self.csr`` is the registered graph), "given" keeps
    the given ids (``self.new_id`` = None)."""
    name = "hits"

    def __init__(self, ctx, n=20_000_000, e=60_000_000, iters=HITS_ITERS, graph=None, vertex_order="degree", **kw):
        super().__init__(ctx, **kw)
        self.n, self.iters = n, iters
        if self.share is not None and graph is None:  # the registered graph of the program shared
            graph, self.new_id = self.share.csr, self.share.new_id
        else:
            if graph is None:
                graph = synth.powerlaw_graph(self.seed, n, e, device=None if ctx.backend == "record" else "auto")
            self.new_id = None
            if vertex_order == "degree":
                graph, self.new_id = degree_order(graph, device=None if ctx.backend == "record" else "auto")
        self.csr = graph
        rp, ci, rpt, cit = graph
        self.e = int(rp[-1])
        stream = self.streaming
        for name, arr in (("rp", rp), ("ci", ci), ("rpt", rpt), ("cit", cit)):
            self.alloc(name, max(1, arr.size), torch.int32)
            if arr.size:
                self.upload(name, arr)
        self.alloc("a1", n, torch.float32, mirror=stream)
        self.alloc("h1", n, torch.float32, mirror=stream)
        gs = spmv_nz_grid(self.e + n)  # padded items <= E + N
        ob = 4 * n + 16 + 12 * SPMV_WARPS * gs  # y + SpmvWs (3 words per warp)
        self.alloc("a2", 0, None, nbytes=ob)
        self.alloc("h2", 0, None, nbytes=ob)
        # row structure of A and A^T re-encoded for the non-zero-split SpMV,
        # once, when the graph is registered
        if self.share is not None and "plan" in self.share.t:
            self.plans = self.share.plans
        else:
            self.plans = (spmv_pad_plan(rp, ci), spmv_pad_plan(rpt, cit))
        for name, arr in (("plan", self.plans[0]), ("plant", self.plans[1])):
            self.alloc(name, arr.size, torch.int32)
            self.upload(name, arr)
        self.alloc_red("an")
        self.alloc_red("hn")
        self.inputs, self.sinks = ["a1", "h1"], ["a1", "h1"]
        a = self.a
        P = ctx.prepare
        ge = grid_1d(n, 256, 4)
        gr = min(grid_1d(n, 256, 8), 1024)
        self.it = [
            P("spmv", gs, 256, [a["rpt"], a["cit"], a["plant"], a["h1"], a["a2"], n]),  # a2 = A^T h1
            P("spmv", gs, 256, [a["rp"], a["ci"], a["plan"], a["a1"], a["h2"], n]),      # h2 = A a1
            P("l2norm", gr, 256, [a["a2"], a["an"], n]),
            P("l2norm", gr, 256, [a["h2"], a["hn"], n]),
            P("divide", ge, 256, [a["a2"], a["an"], a["a1"], n]),
            P("divide", ge, 256, [a["h2"], a["hn"], a["h1"], n]),
        ]

    def _inputs(self, set_index=0):
        v = 1.0 / math.sqrt(self.n) if self.n else 0.0
        for name in ("a1", "h1"):
            if not self.record:
                self.t[name].fill_(v)
            if name in self.mirror:
                self.mirror[name].fill_(v)

    def restart(self):
        """a1 = h1 = 1/sqrt(N) again before a run (host writes, as in the
        golden HITS DAG): stream mode rewrites the pinned mirrors (uploaded
        by the run's prefetches), resident mode writes the device arrays
        through dagrt_host_write, so every run is the same K-iteration DAG
        from the same start vector instead of continuing the last run."""
        v = 1.0 / math.sqrt(self.n) if self.n else 0.0
        if self.record:
            return
        super().restart()  # UM mode: the inputs' pages back to the host
        if self.mode == "stream":
            for name in ("a1", "h1"):
                self.mirror[name].fill_(v)
            return
        if getattr(self, "_init", None) is None:
            self._init = torch.full((max(1, self.n),), v, dtype=torch.float32, pin_memory=True)
        for name in ("a1", "h1"):
            self.ctx.host_write(self.a[name], self._init.data_ptr(), 0, 4 * self.n)

    def launch_sequence(self):
        return [L for _ in range(self.iters) for L in self.it]

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        prev = {"a1": [io["a1"]] if io else [], "h1": [io["h1"]] if io else []}
        sa = sh = sma = smh = da = dh = None
        for k in range(self.iters):
            L = self.it
            # a2 = A^T h1 needs h1 (div_h of the previous iteration) and the
            # previous readers of a2 (sum_a, div_a) to be done.
            sa = g.kernel(L[0], ([dh] if dh is not None else prev["h1"]) + ([da] if da is not None else []))
            sh = g.kernel(L[1], ([da] if da is not None else prev["a1"]) + ([dh] if dh is not None else []))
            sma = g.kernel(L[2], [sa] + ([da] if da is not None else []))
            smh = g.kernel(L[3], [sh] + ([dh] if dh is not None else []))
            da = g.kernel(L[4], [sa, sh, sma])
            dh = g.kernel(L[5], [sa, sh, smh])
        self.graph_sinks(g, {"a1": da, "h1": dh})
        g.instantiate()
        return g

    def kernel_bytes(self):
        n, e = self.n, self.e
        sp = 4 * (n + 1) + 4 * e + 4 * n + 4 * n
        out = {}
        for k in range(self.iters):
            out.update({f"spmv_a{k}": sp, f"spmv_h{k}": sp, f"l2norm_a{k}": 4 * n,
                        f"l2norm_h{k}": 4 * n, f"divide_a{k}": 8 * n, f"divide_h{k}": 8 * n})
        return out

    def vec(self, name):
        return self.t[name][: 4 * self.n].view(torch.float32) if self.t[name].dtype == torch.uint8 \
            else self.t[name]


def dl_shapes(h, w):
    h1, w1 = (h + 1) // 2, (w + 1) // 2
    h2, w2 = h1 // 2, w1 // 2
    h3, w3 = (h2 + 1) // 2, (w2 + 1) // 2
    return (h1, w1), (h2, w2), (h3, w3)


class DeepLearning(Program):
    """Two-branch CNN projecting two images, merged by a dense layer (L887-891)."""
    name = "dl"

    def __init__(self, ctx, h=16384, w=16384, **kw):
        super().__init__(ctx, **kw)
        self.h, self.w = h, w
        (h1, w1), (h2, w2), (h3, w3) = dl_shapes(h, w)
        self.shapes = ((h1, w1), (h2, w2), (h3, w3))
        stream = self.streaming
        nz = 2 * h3 * w3 * 16
        self.alloc("x", h * w, torch.float32, mirror=stream)
        self.alloc("y", h * w, torch.float32, mirror=stream)
        self.alloc("w1", 72, torch.float32)
        self.alloc("w2", 16 * 72, torch.float32)
        self.alloc("wd", max(1, nz), torch.float32)
        for b in ("x", "y"):
            self.alloc(f"c1{b}", max(1, h1 * w1 * 8), torch.float32)
            # + 8 floats: a row-staged conv2 reads one pixel past the last row when W2 is odd
            self.alloc(f"p{b}", h2 * w2 * 8 + 8, torch.float32)
            self.alloc(f"c2{b}", max(1, h3 * w3 * 16), torch.float32)
        self.alloc("z", max(1, nz), torch.float32)
        self.alloc_red("r")
        self.inputs, self.sinks = ["x", "y"], ["r"]
        self.nz = nz
        a = self.a
        P = ctx.prepare
        # conv grids: x = column pairs / 256, y = output rows (<= 65535, kernels loop)
        x1b = max(1, -(-((w1 + 1) // 2) // 256))
        # blocks loop over output row PAIRS ("conv1" = k_conv1_r2b3), ~32 blocks per SM
        g1 = (x1b, max(1, min((h1 + 1) // 2, -(-32 * SMS // x1b))))
        gp = grid_1d(h2 * w2 * 2, 256)
        x2b = max(1, -(-((w3 + 1) // 2) // 256))
        g2 = (x2b, max(1, min(h3, -(-8 * SMS // x2b))))
        gc = grid_1d(nz // 4 + 1, 256)
        self.L = [
            P("conv1", g1, 256, [a["x"], a["w1"], a["c1x"], h, w]),
            P("conv1", g1, 256, [a["y"], a["w1"], a["c1y"], h, w]),
            P("pool", gp, 256, [a["c1x"], a["px"], h1, w1]),
            P("pool", gp, 256, [a["c1y"], a["py"], h1, w1]),
            P("conv2", CONV2_GRID, CONV2_THREADS, [a["px"], a["w2"], a["c2x"], h2, w2], smem=CONV2_SMEM),
            P("conv2", CONV2_GRID, CONV2_THREADS, [a["py"], a["w2"], a["c2y"], h2, w2], smem=CONV2_SMEM),
            P("concat", gc, 256, [a["c2x"], a["c2y"], a["z"], nz // 2, nz // 2]),
            P("dot", min(gc, 1024), 256, [a["z"], a["wd"], a["r"], nz]),
        ]

    def _inputs(self, set_index=0):
        spec = synth.spec_dl(self.h, self.w)
        self.fill("x", spec["x"], set_index)
        self.fill("y", spec["y"], set_index)
        for k in ("w1", "w2", "wd"):
            self.fill(k, spec[k], 0)

    def graph(self):
        g = self.ctx.graph()
        io = self.graph_io(g)
        L = self.L
        cx = g.kernel(L[0], [io["x"]] if io else [])
        cy = g.kernel(L[1], [io["y"]] if io else [])
        px = g.kernel(L[2], [cx])
        py = g.kernel(L[3], [cy])
        c2x = g.kernel(L[4], [px])
        c2y = g.kernel(L[5], [py])
        cc = g.kernel(L[6], [c2x, c2y])
        dt = g.kernel(L[7], [cc])
        self.graph_sinks(g, {"r": dt})
        g.instantiate()
        return g

    def kernel_bytes(self):
        h, w = self.h, self.w
        (h1, w1), (h2, w2), (h3, w3) = self.shapes
        c1 = 4 * h * w + 32 * h1 * w1
        pl = 32 * h1 * w1 + 32 * h2 * w2
        c2 = 32 * h2 * w2 + 64 * h3 * w3
        return {"conv1_x": c1, "conv1_y": c1, "pool_x": pl, "pool_y": pl, "conv2_x": c2,
                "conv2_y": c2, "concat": 8 * self.nz, "dot": 8 * self.nz}

    def result(self):
        return float(self.t["r"][:4].view(torch.float32)[0])
