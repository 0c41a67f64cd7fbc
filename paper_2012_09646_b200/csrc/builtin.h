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

// Launch contract of a built-in kernel, checked by the scheduler before the
// launch becomes a vertex (dagrt_launch / _raw / dagrt_graph_add_kernel):
// array sizes against the scalar shape arguments, grid / block / dynamic
// shared memory against what the kernel assumes.  A violation returns
// DAGRT_EINVAL with the message instead of an out-of-bounds access or a
// hang on the device.
struct LaunchCheck {
  const uint64_t* vals;   // marshalled arguments in C-ABI order (device pointers, scalars)
  const uint64_t* bytes;  // registered size of each array argument (0 for scalars)
  int nargs;
  uint32_t grid[3], block[3], smem;
  bool real;              // CUDA backend (false: the recording backend, no device queries)
  int64_t i(int k) const { return (int64_t)vals[k]; }
  int32_t i32(int k) const { return (int32_t)(uint32_t)vals[k]; }
  uint64_t nthreads() const { return (uint64_t)block[0] * block[1] * block[2]; }
};
typedef const char* (*ValidateFn)(const LaunchCheck& L);  // nullptr = OK, else why not

struct Builtin {
  const char* name;
  const void* fn;
  const char* signature;
  int32_t flags;
  int32_t smem_max;        // > 0: opt in to this much dynamic shared memory (bytes)
  PrelaunchFn prelaunch;   // optional (nullptr)
  ValidateFn validate;     // optional (nullptr)
};

// Shared checks for validators
inline bool fits(const LaunchCheck& L, int arg, uint64_t need) { return L.bytes[arg] >= need; }
// scalar-reduction output (RedOut, kcommon.cuh): 8 bytes + one fp64 partial per block, <= 1024 blocks
inline const char* check_reduction(const LaunchCheck& L, int out_arg) {
  if (L.grid[0] > 1024 || L.grid[1] != 1 || L.grid[2] != 1) return "reduction grid must be 1-D with <= 1024 CTAs";
  if (L.block[0] % 32 || L.block[0] > 1024 || L.block[1] != 1 || L.block[2] != 1)
    return "reduction block must be 1-D, a multiple of 32, <= 1024";
  if (!fits(L, out_arg, 8 + 8ull * L.grid[0])) return "reduction output smaller than 8 + 8 * grid bytes";
  return nullptr;
}

int register_builtins(const Builtin* table, int n);  // returns n
int builtin_count();
const Builtin* builtin_at(int i);

// Built-ins compiled into ANOTHER shared library (the experimental variants,
// libdagrt_exp.so) live in that library's own (static) CUDA runtime: the
// scheduler cannot resolve their host stubs itself.  Such a library registers
// its table with its own resolver, which returns the CUfunction of a stub of
// that library (cudaGetFuncBySymbol there); the scheduler launches it with
// cuLaunchKernel and applies the dynamic shared memory opt-in with the driver.
typedef int (*ResolveFn)(const void* stub, void** cufunc);
int register_builtins_ext(const Builtin* table, int n, ResolveFn resolve);
ResolveFn builtin_resolver(const void* stub);  // nullptr: a stub of libdagrt.so itself

// Scheduler-internal kernel (kernels_runtime.cu): small host reads through
// mapped pinned memory; args (src, dst_mapped_dev, n, flag_dev, seq).
const void* read_mapped_kernel();

}  // namespace dagrt

#define DAGRT_REGISTER_BUILTINS(tbl) \
  static int dagrt_reg_##tbl = ::dagrt::register_builtins(tbl, (int)(sizeof(tbl) / sizeof(tbl[0])))
