"""Integer work beside the FP64 pipe (tools/fp64_issue_lab.cu): cycles per
DFMA warp-instruction per SM sub-partition with 0/8/16/32 integer ops per 8
DFMAs.    python tools/fp64_issue_lab.py"""
import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    so = os.path.join(HERE, "libfp64lab.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "fp64_issue_lab.cu")])
    L = C.CDLL(so)
    iters, mhz = 20000, 1965.0
    out = {}
    for v, nint in enumerate((0, 8, 16, 32)):
        ms = C.c_float()
        rc = L.fp64_issue_lab(v, iters, C.byref(ms))
        warps_per_smsp = 296 * 8 / (148 * 4)
        dfma_instr = iters * 8 * warps_per_smsp  # DFMA warp-instructions per SMSP
        cyc = ms.value * 1e-3 * mhz * 1e6
        out[f"int{nint}"] = {"rc": rc, "ms": ms.value, "cycles_per_dfma_instr": cyc / dfma_instr,
                             "int_instr_per_dfma": nint / 8}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
