// Registry of the built-in sm_100a benchmark kernels linked into libdagrt.so.
// Each kernels_*.cu file registers its __global__ functions with the
// signature the DAG scheduler uses to infer dependencies (include/dagrt.h).
#pragma once
#include <cstdint>

namespace dagrt {

enum : int32_t { KF_NONE = 0, KF_COOPERATIVE = 1 };

struct Builtin {
  const char* name;
  const void* fn;
  const char* signature;
  int32_t flags;
  int32_t smem_max;  // > 0: opt in to this much dynamic shared memory (bytes)
};

int register_builtins(const Builtin* table, int n);  // returns n
int builtin_count();
const Builtin* builtin_at(int i);

// Scheduler-internal kernel (kernels_runtime.cu): small host reads through
// mapped pinned memory; args (src, dst_mapped_dev, n, flag_dev, seq).
const void* read_mapped_kernel();

}  // namespace dagrt

#define DAGRT_REGISTER_BUILTINS(tbl) \
  static int dagrt_reg_##tbl = ::dagrt::register_builtins(tbl, (int)(sizeof(tbl) / sizeof(tbl[0])))
