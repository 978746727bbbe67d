// Device copy of synth.gen_item (synth/__init__.py): the seeded synthetic KV
// values of one item, [L][h1-h0][T][D] 16-bit.  Input generation only — no
// HA-RAG arithmetic.  Same integer hash and fp32 operations (explicit _rn
// intrinsics, no contraction) as the numpy copy; tests cross-check the two.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen_item_kernel(uint64_t seed, uint32_t L, uint32_t H, uint32_t T, uint32_t D, uint32_t h0,
                                uint32_t Hs, uint64_t item, int kind, int fp16, uint16_t* dst) {
  const uint64_t n = (uint64_t)L * Hs * T * D;
  const float k_unit = (float)(4.0 / 37837.0), v_unit = (float)(2.5 / 37837.0);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = i % D;
    uint64_t r = i / D;
    const uint64_t t = r % T;
    r /= T;
    const uint64_t hs = r % Hs;
    const uint64_t l = r / Hs;
    const uint64_t gidx = ((((item * L + l) * H + (h0 + hs)) * T + t) * D + d);
    const uint64_t u = splitmix64(seed ^ gidx);
    const int64_t b = (int64_t)((u & 0xFFFF) + ((u >> 16) & 0xFFFF) + ((u >> 32) & 0xFFFF) + (u >> 48)) - 131070;
    float x;
    if (kind == 0) {
      x = __fmul_rn((float)b, k_unit);
      if (d % 16 == 0) x = __fmul_rn(x, 2.5f);
      x = fminf(fmaxf(x, -24.875f), 24.875f);
    } else {
      x = __fmul_rn((float)b, v_unit);
      x = fminf(fmaxf(x, -9.9375f), 9.9375f);
    }
    dst[i] = fp16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
}

}  // namespace

extern "C" int hrs_gen_item(uint64_t seed, uint32_t L, uint32_t H, uint32_t T, uint32_t D, uint32_t h0, uint32_t h1,
                            uint32_t doc, uint32_t kind, uint32_t alias_R, int fp16, uint32_t reserved, void* dst,
                            void* stream) {
  (void)reserved;
  if (h1 <= h0 || h1 > H || kind > 1 || !dst) return 1;
  const uint32_t adoc = alias_R ? doc % alias_R : doc;
  const uint64_t item = 2ull * adoc + kind;
  gen_item_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(seed, L, H, T, D, h0, h1 - h0, item, (int)kind, fp16,
                                                            (uint16_t*)dst);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
