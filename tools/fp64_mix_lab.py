"""FP64-side instruction costs (tools/fp64_mix_lab.cu): cycles per
warp-instruction per SM sub-partition, 16 warps per SM, 8 independent
chains per thread.    python tools/fp64_mix_lab.py"""
import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ["dfma_reg", "dfma_cbank", "dmul", "dadd", "mufu_rcp64h", "i2f_f64_plus_dadd",
         "8dfma_plus_1rcp64h", "8dfma_plus_1rcp_f32"]


def main():
    so = os.path.join(HERE, "libfp64mix.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "fp64_mix_lab.cu")])
    L = C.CDLL(so)
    iters, mhz = 20000, 1965.0
    out = {}
    for v, name in enumerate(NAMES):
        ms = C.c_float()
        rc = L.fp64_mix_lab(v, iters, C.byref(ms))
        warps_per_smsp = 296 * 8 / (148 * 4)
        instr = iters * 8 * warps_per_smsp
        out[name] = {"rc": rc, "ms": ms.value, "cycles_per_warp_instr": ms.value * 1e-3 * mhz * 1e6 / instr}
        if v >= 6:  # per iteration: 8 DFMA + 1 extra; report cycles per 8-DFMA group
            out[name]["cycles_per_8dfma_group"] = ms.value * 1e-3 * mhz * 1e6 / (iters * warps_per_smsp)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
