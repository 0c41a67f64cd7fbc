// Experimental built-in variants (libdagrt_exp.so): the tuning alternatives
// measured against the product kernels (tools/*_variants.py, profiles/) and
// kept tested, but not part of the product library.  They are compiled into
// their own shared library, loaded on request (dagrt.load_experimental()),
// and register into the same built-in registry with this library's own
// kernel resolver (builtin.h register_builtins_ext): its CUDA runtime is not
// libdagrt.so's.
#pragma once
#include <cuda_runtime.h>

#include "../builtin.h"

namespace dagrt {
namespace expv {
inline int resolve(const void* stub, void** f) {
  cudaFunction_t cf = nullptr;
  if (cudaGetFuncBySymbol(&cf, stub) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  *f = (void*)cf;
  return 0;
}
}  // namespace expv
}  // namespace dagrt

#define DAGRT_REGISTER_EXP(tbl)                                                                       \
  static int dagrt_exp_reg_##tbl =                                                                    \
      ::dagrt::register_builtins_ext(tbl, (int)(sizeof(tbl) / sizeof(tbl[0])), ::dagrt::expv::resolve)
