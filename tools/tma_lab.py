"""TMA throughput for the conv2 input patterns (tools/tma_lab.cu), full DL
conv2 shape (4096 x 4096 x 8 fp32):
    python tools/tma_lab.py"""
import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import torch
    so = os.path.join(HERE, "libtmalab.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "tma_lab.cu"), "-lcuda"])
    L = C.CDLL(so)
    L.tma_lab.restype = C.c_float
    L.tma_lab.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int]
    H2 = W2 = 4096
    x = torch.rand(H2 * W2 * 8, device="cuda")
    out = {}
    for mode, name in ((0, "9 strided boxes (product)"), (1, "9 contiguous boxes"), (2, "6 contiguous row boxes")):
        for st in (4, 6):
            ms = L.tma_lab(mode, st, x.data_ptr(), H2, W2, 10)
            out[f"{name} S={st}"] = {"us": ms * 1e3}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
