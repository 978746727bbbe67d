// Exhaustive check (test infrastructure) of the division-free INT8 code arithmetic used by
// quantize.cu: for every finite 16-bit magnitude a (the group absmax, bf16 or fp16) and every
// 16-bit value x with |x| <= a, compare
//   s  = RN(a / 127)                  (IEEE)   vs  div127(a)          (Markstein correction)
//   q  = RN(x / s)                    (IEEE)   vs  markstein(x, s, y), y = RN(1/s)
// Prints "mismatches <n> pairs <m>"; exit code 0 iff n == 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tests/csrc/markstein_check tests/csrc/markstein_check.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdint>

__device__ float to_f32(uint32_t b, int fp16) {
  return fp16 ? __half2float(__ushort_as_half((unsigned short)b)) : __uint_as_float(b << 16);
}
__device__ float div127(float a) {
  const float y = 0.007874015718698501587f;
  if (a < 7.8886090522101181e-31f) return __fdiv_rn(a, 127.f);
  const float q0 = __fmul_rn(a, y);
  const float r = __fmaf_rn(-q0, 127.f, a);
  return __fmaf_rn(r, y, q0);
}
__device__ float markstein(float x, float s, float y) {
  const float q0 = __fmul_rn(x, y);
  const float r = __fmaf_rn(-q0, s, x);
  return __fmaf_rn(r, y, q0);
}

__device__ unsigned int g_nrec;
__device__ uint32_t g_rec[64];
__global__ void check(int fp16, uint32_t top, unsigned long long* bad, unsigned long long* pairs) {
  const uint32_t a_bits = blockIdx.x + 1;  // 1 .. top
  if (a_bits > top) return;
  const float a = to_f32(a_bits, fp16);
  const float s_ref = __fdiv_rn(a, 127.f);
  const float s = div127(a);
  unsigned long long nb = (__float_as_uint(s) != __float_as_uint(s_ref)), np = 0;
  const float y = __fdiv_rn(1.f, s_ref);
  const bool normal = s_ref >= 8.0779356e-28f && s_ref <= 4.2535296e+37f;  // 2^-90 .. 2^125: the residual cannot underflow
  for (uint32_t xb = threadIdx.x; xb <= a_bits; xb += blockDim.x) {
    const float x = to_f32(xb, fp16);
    for (int sign = 0; sign < 2; ++sign) {
      const float xs = sign ? -x : x;
      const float ref = __fdiv_rn(xs, s_ref);
      if (normal) {
        const float q = markstein(xs, s_ref, y);
        if (__float2int_rn(q) != __float2int_rn(ref)) {
          ++nb;
          const unsigned k = atomicAdd(&g_nrec, 1u);
          if (k < 16) g_rec[4 * k] = a_bits, g_rec[4 * k + 1] = xb | (sign << 16), g_rec[4 * k + 2] = __float_as_uint(q),
                                     g_rec[4 * k + 3] = __float_as_uint(ref);
        }
      }
      ++np;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(pairs, np);
}

int main() {
  unsigned long long *bad, *pairs;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&pairs, 8);
  unsigned long long total_bad = 0, total_pairs = 0;
  for (int fp16 = 0; fp16 < 2; ++fp16) {
    *bad = *pairs = 0;
    const uint32_t top = fp16 ? 0x7BFF : 0x7F7F;
    check<<<top, 256>>>(fp16, top, bad, pairs);
    cudaDeviceSynchronize();
    printf("%s: mismatches %llu pairs %llu\n", fp16 ? "fp16" : "bf16", *bad, *pairs);
    unsigned n = 0;
    uint32_t rec[64];
    cudaMemcpyFromSymbol(&n, g_nrec, 4);
    cudaMemcpyFromSymbol(rec, g_rec, sizeof(rec));
    for (unsigned i = 0; i < n && i < 16; ++i)
      printf("  a=0x%04x x=0x%05x q=%08x ref=%08x\n", rec[4 * i], rec[4 * i + 1], rec[4 * i + 2], rec[4 * i + 3]);
    unsigned z = 0;
    cudaMemcpyToSymbol(g_nrec, &z, 4);
    total_bad += *bad;
    total_pairs += *pairs;
  }
  printf("mismatches %llu pairs %llu err %s\n", total_bad, total_pairs, cudaGetErrorString(cudaGetLastError()));
  return total_bad == 0 ? 0 : 1;
}
