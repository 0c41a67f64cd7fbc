"""The product SpMV (k_spmv_nz: non-zero split, row structure re-encoded at
graph registration) on hand-made CSR shapes that stress its edge cases,
against the oracle's SpMV (oracle/hits.py): rows spanning
many warp ranges (one giant row; a giant first / last row), long runs of empty
rows before, between and after the non-empty ones, an all-empty matrix,
ragged last chunks, and grids from one warp to more warps than chunks.  Every
case also runs twice (the arrival counters must reset) and must be
bit-identical run to run."""
import numpy as np
import pytest
import torch

import synth
from oracle import hits as ohits
from paper_2012_09646_b200 import dagrt as D
from paper_2012_09646_b200.programs.hits_dl import SPMV_WARPS, spmv_nz_plan, spmv_pad_plan

from oracle_checks import assert_close

pytestmark = pytest.mark.gpu


def csr_from_degrees(deg, n, seed):
    rng = np.random.default_rng(seed)
    rp = np.zeros(len(deg) + 1, np.int64)
    rp[1:] = np.cumsum(deg)
    ci = np.concatenate([np.sort(rng.choice(n, d, replace=d > n)) for d in deg]) if rp[-1] else \
        np.zeros(0, np.int64)
    return rp.astype(np.int32), ci.astype(np.int32)


CASES = {
    "giant_single_row": ([0, 0, 200_000, 0, 0], 300_000),
    "giant_first_row": ([150_000] + [1, 0, 2, 0, 0, 3] * 2000, 50_000),
    "giant_last_row": ([0, 1] * 3000 + [0] * 777 + [90_001], 40_000),
    "all_empty": ([0] * 1000, 1000),
    "one_nonzero": ([0] * 500 + [1] + [0] * 499, 1000),
    "ragged_short": ([1, 2, 3, 0, 4] * 1001 + [5], 7000),
    "exact_chunks": ([4] * 32 * 40, 5000),
    # every 4-item lane holds a row start, rows spanning two lanes (spmv_pad2's
    # one-shuffle path) / some lanes inside a row (the full scan)
    "short_rows": ([1, 2, 2, 1, 3] * 3000, 9000),
    "lane_spanning": ([5, 1, 6, 2] * 2000, 8000),
}


@pytest.fixture(scope="module")
def ctx():
    c = D.Context(device=0)
    yield c
    c.close()


def run_nz(ctx, rp, ci, x, grid, tag, kernel="spmv"):
    n = len(rp) - 1
    plan = spmv_nz_plan(rp) if kernel == "spmv_nz" else spmv_pad_plan(rp, ci)
    ob = 4 * n + 16 + 12 * SPMV_WARPS * grid
    if kernel == "spmv":  # padded items: 4 * N more than E at most
        pass
    t = {"rp": torch.from_numpy(rp).cuda(), "ci": torch.from_numpy(ci if ci.size else np.zeros(4, np.int32)).cuda(),
         "plan": torch.from_numpy(plan).cuda(), "x": torch.from_numpy(x).cuda(),
         "y": torch.full((ob // 4 + 1,), float("nan"), device="cuda")}
    t["y"][n:] = 0.0  # workspace zeroed once by the allocator (as in the programs)
    torch.cuda.synchronize()
    A = [ctx.register_tensor(f"{tag}_{k}", v) for k, v in t.items()]
    outs = []
    for _ in range(2):
        ctx.launch(kernel, grid, 256, *A, n)
        ctx.sync()
        outs.append(t["y"][:n].clone())
    for a in A:
        ctx.unregister(a)
    return outs


@pytest.mark.parametrize("kernel", ["spmv", "spmv_nz", "spmv_pad2", "spmv_pad2b3", "spmv_ws", "spmv_pad_l2", "spmv_tma4", "spmv_tma8"])
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("grid", [1, 7, 148 * 6])
def test_spmv_nz_edge_shapes(ctx, exp, case, grid, kernel):
    deg, ncols = CASES[case]
    rp, ci = csr_from_degrees(deg, ncols, 1)
    n = len(deg)
    x = np.random.default_rng(2).random(max(n, ncols)).astype(np.float32)
    # columns index x of length max(n, ncols): square-ish padding of the matrix
    y1, y2 = run_nz(ctx, rp, ci, x, grid, f"{case}_{grid}_{kernel}", kernel)
    assert torch.equal(y1, y2)
    ref = ohits.spmv(rp, ci, x.astype(np.float64))
    assert_close(y1.cpu().numpy(), ref, case)


@pytest.mark.parametrize("kernel", ["spmv", "spmv_nz", "spmv_pad2", "spmv_pad2b3", "spmv_ws", "spmv_pad_l2", "spmv_tma4", "spmv_tma8"])
@pytest.mark.parametrize("n,e,seed", [(10, 30, 1), (5000, 15000, 3), (300_000, 900_000, 11)])
def test_spmv_nz_powerlaw(ctx, exp, n, e, seed, kernel):
    rp, ci, _, _ = synth.powerlaw_graph(seed, n, e, device="auto")
    x = np.random.default_rng(seed).random(n).astype(np.float32)
    for grid in (3, 148 * 6):
        y1, y2 = run_nz(ctx, rp, ci, x, grid, f"pl{n}_{grid}_{kernel}", kernel)
        assert torch.equal(y1, y2)
        assert_close(y1.cpu().numpy(), ohits.spmv(rp, ci, x.astype(np.float64)), (n, grid))
