"""Cycles per tcgen05.mma (M=128) by kind, N and A source (tools/mma_lab.cu).
    python tools/mma_lab.py"""
import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    so = os.path.join(HERE, "libmmalab.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "mma_lab.cu")])
    L = C.CDLL(so)
    out = {}
    reps = 256
    for kind, kn in ((0, "tf32"), (1, "bf16")):
        for ts in (0, 1):
            for n in (16, 32, 48, 64, 128, 256):
                h = (C.c_longlong * 2)()
                rc = L.mma_lab(kind, ts, n, reps, h)
                out[f"{kn}_{'TS' if ts else 'SS'}_N{n}"] = {"rc": rc, "issue_cyc_per_mma": h[0] / reps,
                                                            "total_cyc_per_mma": h[1] / reps}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
