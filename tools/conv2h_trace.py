"""Per-tile hand-off times of the warp-specialised conv2 on CTA 0 (tools/conv2h_trace.cu).
    python tools/conv2h_trace.py"""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
NAMES = ["prod_slot", "prod_issued", "mma_loready", "mma_accempty", "mma_issued", "split_full", "split_bufok",
         "split_done", "epi_acc", "epi_done"]


def main():
    import numpy as np
    import torch
    so = os.path.join(HERE, "libc2htrace.so")
    csrc = os.path.join(os.path.dirname(HERE), "paper_2012_09646_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", f"-I{csrc}", "-o", so,
                           os.path.join(HERE, "conv2h_trace.cu"), "-lcuda"])
    L = C.CDLL(so)
    H2 = W2 = 4096
    x = torch.rand(H2 * W2 * 8 + 8, device="cuda")
    w = torch.rand(16 * 72, device="cuda") - 0.5
    out = torch.empty(((H2 + 1) // 2) * ((W2 + 1) // 2) * 16, device="cuda")
    tr = (C.c_longlong * 640)()
    rc = L.conv2h_trace(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(out.data_ptr()), H2, W2, tr)
    assert rc == 0, rc
    t = np.array(tr[:], dtype=np.int64).reshape(10, 64)
    t0 = t[0, 0]
    t = t - t0
    print("tile " + " ".join(f"{n:>12s}" for n in NAMES))
    for i in range(0, 40):
        print(f"{i:4d} " + " ".join(f"{v:12d}" for v in t[:, i]))
    d = np.diff(t, axis=1)[:, 8:40].mean(axis=1)
    print("mean cycles between consecutive tiles per point:", dict(zip(NAMES, np.round(d))))


if __name__ == "__main__":
    main()
