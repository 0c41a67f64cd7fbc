"""Bounds of the HITS SpMV on the real graph (tools/spmv_lab.cu):
gather-only throughput per cache operator, stream-only, gathers with the K
most frequent columns staged in shared memory, next to the product k_spmv.

    python tools/spmv_lab.py [--out gpurun_out/spmv_lab.json]
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def build():
    so = os.path.join(HERE, "libspmvlab.so")
    src = os.path.join(HERE, "spmv_lab.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", so, src])
    L = C.CDLL(so)
    L.lab_time.restype = C.c_float
    L.lab_time.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                           C.c_longlong, C.c_int, C.c_int]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=20_000_000)
    ap.add_argument("--e", type=int, default=60_000_000)
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    L = build()
    t0 = time.time()
    rp, ci, rpt, cit = synth.powerlaw_graph(synth.BASE_SEED, args.n, args.e, device="auto")
    res = {"graph_s": time.time() - t0, "n": args.n, "e": int(rp[-1])}
    n, E = args.n, int(rp[-1])
    dci = torch.from_numpy(ci).cuda()
    x = torch.rand(n, device="cuda")
    out = torch.zeros(16, device="cuda")
    g = 148 * 8
    names = {0: "gather_ldg", 1: "gather_nc_noalloc", 2: "gather_cg", 3: "gather_evict_last", 4: "stream_only"}
    for w, nm in names.items():
        res[nm + "_us"] = 1e3 * L.lab_time(w, dci.data_ptr(), None, None, 0, x.data_ptr(), out.data_ptr(), E, g, 10)
    cnt = np.bincount(ci, minlength=n)
    order = np.argsort(-cnt, kind="stable")
    for K in (16384, 32768, 49152):
        hubs = order[:K].astype(np.int32)
        slot = np.full(n, 0, np.int64)
        slot[hubs] = np.arange(1, K + 1)
        s = slot[ci]
        ci2 = np.where(s > 0, -s, ci).astype(np.int32)
        dci2 = torch.from_numpy(ci2).cuda()
        dh = torch.from_numpy(hubs).cuda()
        res[f"gather_hub{K}_us"] = 1e3 * L.lab_time(5, None, dci2.data_ptr(), dh.data_ptr(), K, x.data_ptr(),
                                                    out.data_ptr(), E, 148, 10)
        res[f"hub{K}_coverage"] = float((s > 0).mean())
        del dci2
    for K in (8192, 32768, 65536, 131072, 262144):
        hot = np.zeros(n, bool)
        hot[order[:K]] = True
        ci3 = np.where(hot[ci], ci | np.int32(-2**31), ci).astype(np.int32)
        dci3 = torch.from_numpy(ci3).cuda()
        for w, nm in ((6, "split_noalloc"), (7, "split_evictfirst"), (9, "split_noalloc_ci_ef"),
                      (10, "split_evictfirst_ci_ef")):
            res[f"{nm}{K}_us"] = 1e3 * L.lab_time(w, None, dci3.data_ptr(), None, 0, x.data_ptr(),
                                                  out.data_ptr(), E, g, 10)
        res[f"hot{K}_coverage"] = float(hot[ci].mean())
        del dci3
    res["gather_ci_evictfirst_us"] = 1e3 * L.lab_time(8, dci.data_ptr(), None, None, 0, x.data_ptr(),
                                                     out.data_ptr(), E, g, 10)
    for gg in (148 * 4, 148 * 16, 148 * 32):
        res[f"gather_ldg_grid{gg}_us"] = 1e3 * L.lab_time(0, dci.data_ptr(), None, None, 0, x.data_ptr(),
                                                         out.data_ptr(), E, gg, 10)
    # the SpMV kernels on the same graph, through the C ABI
    from paper_2012_09646_b200 import dagrt as D
    D.load_experimental()  # the variants live in libdagrt_exp.so
    from paper_2012_09646_b200.programs.hits_dl import spmv_nz_grid, spmv_nz_plan, spmv_out_bytes, spmv_pad_plan
    ctx = D.Context(device=0)
    ob, grid = spmv_out_bytes(n, E)
    gnz = spmv_nz_grid(E)
    ob = max(ob, 4 * n + 16 + 12 * 8 * 148 * 16)
    y = torch.zeros(ob // 4 + 1, device="cuda")
    drp = torch.from_numpy(rp).cuda()
    t1 = time.time()
    plan = spmv_nz_plan(rp)
    res["nz_plan_s"] = time.time() - t1
    dplan = torch.from_numpy(plan).cuda()
    t1 = time.time()
    pplan = spmv_pad_plan(rp, ci)
    res["pad_plan_s"] = time.time() - t1
    dpplan = torch.from_numpy(pplan).cuda()
    torch.cuda.synchronize()
    A = [ctx.register_tensor(k, t) for k, t in (("rp", drp), ("ci", dci), ("plan", dplan), ("x", x), ("y", y))]
    AP = ctx.register_tensor("pplan", dpplan)
    st = torch.cuda.Stream()

    def timeit(Lp):
        for _ in range(3):
            Lp.raw(st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
            for _ in range(10):
                Lp.raw(st.cuda_stream)
            e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / 10 * 1e3

    res["merge_path_spmv_us"] = timeit(ctx.prepare("spmv_merge", grid, 256, [A[0], A[1], A[3], A[4], n]))
    for cps in (4, 6, 8, 12, 16):
        g2 = max(1, min(-(-(-(-E // 128)) // 8), cps * 148))
        res[f"nz_spmv_cps{cps}_us"] = timeit(ctx.prepare("spmv_nz", g2, 256, A + [n]))
        g3 = max(1, min(-(-(-(-(E + n) // 128)) // 8), cps * 148))
        res[f"pad_spmv_cps{cps}_us"] = timeit(ctx.prepare("spmv", g3, 256, [A[0], A[1], AP, A[3], A[4], n]))
    res["nz_spmv_default_grid"] = gnz
    y0 = y[:n].clone()
    ctx.prepare("spmv_merge", grid, 256, [A[0], A[1], A[3], A[4], n]).raw(st.cuda_stream)
    torch.cuda.synchronize()
    res["nz_vs_merge_max_rel_diff"] = float(((y0 - y[:n]).abs() / (y[:n].abs() + 1e-30)).max())
    res["algorithmic_bytes"] = 4 * (n + 1) + 4 * E + 8 * n
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f)


if __name__ == "__main__":
    main()
