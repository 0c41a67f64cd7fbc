// GPU twin of synth/__init__.py: the same counter-based generator, bit for
// bit, so full-size benchmark inputs are drawn directly in HBM.  Input
// generation only -- holds none of the method's arithmetic.  Every floating
// operation is an explicit round-to-nearest intrinsic (no FMA contraction)
// so the values equal numpy's.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr uint64_t G = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t bits(uint64_t key, uint64_t i) {
  uint64_t z = key + (i + 1) * G;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double f64_unit(uint64_t h) {
  return __dmul_rn((double)(h >> 11), 1.1102230246251565e-16);  // 2^-53
}

__global__ void fill(void* out, long long n, int kind, uint64_t key, double a0, double a1,
                     long long idx0) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    uint64_t h = bits(key, (uint64_t)(idx0 + i));
    switch (kind) {
      case 0:  // f32 U[0,1): top 24 bits * 2^-24
        ((float*)out)[i] = __fmul_rn((float)(unsigned)(h >> 40), 5.9604644775390625e-8f);
        break;
      case 1:  // f64 U[lo,hi) = lo + (hi-lo)*u
        ((double*)out)[i] = __dadd_rn(a0, __dmul_rn(__dsub_rn(a1, a0), f64_unit(h)));
        break;
      case 2: {  // int U{0..m-1} = ((h>>32)*m)>>32
        uint64_t m = (uint64_t)a0;
        ((int*)out)[i] = (int)(((h >> 32) * m) >> 32);
        break;
      }
      case 3:  // f32((2u-1)*scale)
        ((float*)out)[i] =
            __double2float_rn(__dmul_rn(__dsub_rn(__dmul_rn(2.0, f64_unit(h)), 1.0), a0));
        break;
    }
  }
}
}  // namespace

extern "C" int synth_fill(void* dev, long long n, int kind, unsigned long long key, double a0,
                          double a1, long long idx0, void* stream) {
  if (n <= 0) return 0;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  fill<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dev, n, kind, key, a0, a1, idx0);
  return (int)cudaGetLastError();
}

extern "C" int synth_sync(void) { return (int)cudaDeviceSynchronize(); }
