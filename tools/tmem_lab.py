"""Checks tcgen05.mma.kind::tf32 with A in tensor memory (tools/tmem_lab.cu)
against A in shared memory and a CPU reference (operands truncated to tf32).
    python tools/tmem_lab.py"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import torch
    so = os.path.join(HERE, "libtmemlab.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "tmem_lab.cu")])
    L = C.CDLL(so)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((128, 72)).astype(np.float32)
    B = rng.standard_normal((16, 72)).astype(np.float32)
    tr = lambda x: (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)  # noqa: E731
    ref = tr(A) @ tr(B).T
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for mode in (0, 1):
        D = torch.zeros(128 * 16, device="cuda")
        rc = L.tmem_lab(mode, C.c_void_p(dA.data_ptr()), C.c_void_p(dB.data_ptr()), C.c_void_p(D.data_ptr()))
        d = D.cpu().numpy().reshape(128, 16).astype(np.float64)
        err = np.abs(d - ref).max() / np.abs(ref).max()
        print(f"mode {mode} ({'A smem' if mode == 0 else 'A tmem'}): rc={rc} max rel err {err:.3e}")
        if err > 1e-5:
            # which permutation of rows/cols would match?
            print("  D[0,:4]", d[0, :4], "ref", ref[0, :4])
    A16 = rng.standard_normal((128, 64)).astype(np.float16)
    B16 = rng.standard_normal((16, 64)).astype(np.float16)
    ref16 = A16.astype(np.float64) @ B16.astype(np.float64).T
    dA16, dB16 = torch.from_numpy(A16).cuda(), torch.from_numpy(B16).cuda()
    D = torch.zeros(128 * 16, device="cuda")
    rc = L.tmem_lab_f16(C.c_void_p(dA16.data_ptr()), C.c_void_p(dB16.data_ptr()), C.c_void_p(D.data_ptr()))
    d = D.cpu().numpy().reshape(128, 16).astype(np.float64)
    print(f"kind::f16 A tmem (2 fp16 per column): rc={rc} max rel err {np.abs(d - ref16).max() / np.abs(ref16).max():.3e}")


if __name__ == "__main__":
    main()
