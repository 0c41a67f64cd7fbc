// Registry of the built-in sm_100a benchmark kernels linked into libdagrt.so.
// Each kernels_*.cu file registers its __global__ functions with the
// signature the DAG scheduler uses to infer dependencies (include/dagrt.h).
#pragma once
#include <cstdint>

namespace dagrt {

enum : int32_t { KF_NONE = 0, KF_COOPERATIVE = 1 };

// Host-side pre-launch hook of a built-in kernel: given the marshalled
// argument values of the C-ABI signature (device pointers, scalars), returns
// one extra pointer-sized value passed to the CUDA kernel BEFORE them (e.g.
// a TMA tensor-map descriptor in device memory built from the pointer and
// shape arguments).  The signature -- and so the DAG -- is unchanged.
typedef int (*PrelaunchFn)(const uint64_t* vals, int nargs, void** extra);

struct Builtin {
  const char* name;
  const void* fn;
  const char* signature;
  int32_t flags;
  int32_t smem_max;        // > 0: opt in to this much dynamic shared memory (bytes)
  PrelaunchFn prelaunch;   // optional (nullptr)
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
