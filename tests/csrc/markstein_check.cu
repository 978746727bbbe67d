// Exhaustive check (test infrastructure) of the division-free INT8 code arithmetic used by
// quantize.cu: for every finite 16-bit magnitude a (the group absmax, bf16 or fp16) and every
// 16-bit value x with |x| <= a, compare
//   s  = RN(a / 127)                  (IEEE)   vs  div127(a)          (Markstein correction)
//   q  = RN(x / s)                    (IEEE)   vs  markstein(x, s, y), y = RN(1/s)
// INT4 (sampled): for 2^36 counter-hashed (x, mn, mx) triples of finite 16-bit values per dtype, half
// of them with x steered next to a quantisation tie, compare
//   q  = rne(RN(u / s))               (IEEE)   vs  rne(markstein2(u, s, y)), u = RN(x - mn),
//   s  = RN(RN(mx - mn) / 15), y = RN(1/s)     (two Markstein corrections, quantize.cu enc_int4_step)
// Scale / reciprocal (exhaustive over fp32 significands): for every d = 1.m * 2^e, e in [-100, 127],
//   RN(d / 15) (IEEE) vs div15(d) (one Markstein correction), and RN(1/d) (IEEE division) vs __frcp_rn(d).
// Prints "mismatches <n> pairs <m>"; exit code 0 iff n == 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tests/csrc/markstein_check tests/csrc/markstein_check.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdint>

__device__ unsigned int g_nrec;
__device__ uint32_t g_rec[64];

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

__device__ float div15(float d) {  // quantize.cu div15 (d >= 2^-100)
  const float y = 0.066666670143604278564f;
  const float q0 = __fmul_rn(d, y);
  const float r = __fmaf_rn(-q0, 15.f, d);
  return __fmaf_rn(r, y, q0);
}
__global__ void check_scale(unsigned long long* bad, unsigned long long* pairs) {
  unsigned long long nb = 0, np = 0;
  const unsigned long long n = 228ull << 23;  // biased exponents 27 (2^-100) .. 254 (2^127)
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float d = __uint_as_float((uint32_t)(((i >> 23) + 27) << 23 | (i & 0x7FFFFF)));
    const float q = div15(d), ref = __fdiv_rn(d, 15.f);
    const float y = __frcp_rn(d), yref = __fdiv_rn(1.f, d);
    if (__float_as_uint(q) != __float_as_uint(ref) || __float_as_uint(y) != __float_as_uint(yref)) {
      ++nb;
      const unsigned k = atomicAdd(&g_nrec, 1u);
      if (k < 16) g_rec[4 * k] = __float_as_uint(d), g_rec[4 * k + 1] = __float_as_uint(q), g_rec[4 * k + 2] = __float_as_uint(ref),
                                 g_rec[4 * k + 3] = __float_as_uint(y) ^ __float_as_uint(yref);
    }
    np += 2;
  }
  atomicAdd(bad, nb);
  atomicAdd(pairs, np);
}

// two corrections: q1 is faithful, q2 = RN(u / s) (Markstein's theorem)
__device__ float markstein2(float u, float s, float y) {
  const float q0 = __fmul_rn(u, y);
  const float q1 = __fmaf_rn(__fmaf_rn(-q0, s, u), y, q0);
  return __fmaf_rn(__fmaf_rn(-q1, s, u), y, q1);
}
__device__ __forceinline__ unsigned long long splitmix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ uint32_t finite16(uint32_t b, int fp16) {  // map 16 random bits to a finite pattern
  const uint32_t top = fp16 ? 0x7BFFu : 0x7F7Fu;
  return (b & 0x8000u) | ((b & 0x7FFFu) % (top + 1));
}
__device__ float from16(uint32_t b, int fp16) { return fp16 ? __half2float(__ushort_as_half((unsigned short)b)) : __uint_as_float(b << 16); }
__device__ uint32_t to16(float v, int fp16) {  // RN to the source dtype
  return fp16 ? (uint32_t)__half_as_ushort(__float2half_rn(v)) : (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
}

__global__ void check_int4(int fp16, unsigned long long n, unsigned long long* bad, unsigned long long* pairs) {
  unsigned long long nb = 0, np = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long h = splitmix(i * 2 + (unsigned long long)fp16);
    float a = from16(finite16((uint32_t)h & 0xFFFFu, fp16), fp16);
    float b = from16(finite16((uint32_t)(h >> 16) & 0xFFFFu, fp16), fp16);
    const float mn = __fadd_rn(fminf(a, b), 0.f), mx = __fadd_rn(fmaxf(a, b), 0.f);
    const float dm = __fsub_rn(mx, mn);
    if (!(dm <= 3.40282347e+38f)) continue;
    const float s = (mx == mn) ? 1.f : __fdiv_rn(dm, 15.f);
    if (!(s >= 8.0779356e-28f && s <= 4.2535296e+37f)) continue;
    float x;
    if ((h >> 32) & 1) {  // x steered to a half-integer quotient k + 1/2, then rounded to the source dtype
      const float k = (float)((h >> 33) % 15) + 0.5f;
      x = from16(to16(__fadd_rn(mn, __fmul_rn(k, s)), fp16), fp16);
      x = fminf(fmaxf(x, mn), mx);
    } else {
      x = from16(finite16((uint32_t)(h >> 40) & 0xFFFFu, fp16), fp16);
      x = fminf(fmaxf(x, mn), mx);
    }
    const float u = __fsub_rn(x, mn);
    const float y = __frcp_rn(s);
    const int ref = __float2int_rn(__fdiv_rn(u, s)), got = __float2int_rn(markstein2(u, s, y));
    if (ref != got) {
      ++nb;
      const unsigned k = atomicAdd(&g_nrec, 1u);
      if (k < 16) g_rec[4 * k] = __float_as_uint(u), g_rec[4 * k + 1] = __float_as_uint(s), g_rec[4 * k + 2] = got,
                                 g_rec[4 * k + 3] = ref;
    }
    ++np;
  }
  atomicAdd(bad, nb);
  atomicAdd(pairs, np);
}

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
  {
    *bad = *pairs = 0;
    check_scale<<<148 * 8, 256>>>(bad, pairs);
    cudaDeviceSynchronize();
    printf("scale div15 / rcp: mismatches %llu values %llu\n", *bad, *pairs);
    unsigned n = 0;
    uint32_t rec[64];
    cudaMemcpyFromSymbol(&n, g_nrec, 4);
    cudaMemcpyFromSymbol(rec, g_rec, sizeof(rec));
    for (unsigned i = 0; i < n && i < 16; ++i)
      printf("  d=%08x q=%08x ref=%08x rcpxor=%08x\n", rec[4 * i], rec[4 * i + 1], rec[4 * i + 2], rec[4 * i + 3]);
    unsigned z = 0;
    cudaMemcpyToSymbol(g_nrec, &z, 4);
    total_bad += *bad;
    total_pairs += *pairs;
  }
  for (int fp16 = 0; fp16 < 2; ++fp16) {
    *bad = *pairs = 0;
    check_int4<<<148 * 8, 256>>>(fp16, 1ull << 36, bad, pairs);
    cudaDeviceSynchronize();
    printf("int4 %s: mismatches %llu triples %llu\n", fp16 ? "fp16" : "bf16", *bad, *pairs);
    unsigned n = 0;
    uint32_t rec[64];
    cudaMemcpyFromSymbol(&n, g_nrec, 4);
    cudaMemcpyFromSymbol(rec, g_rec, sizeof(rec));
    for (unsigned i = 0; i < n && i < 16; ++i)
      printf("  u=%08x s=%08x got=%d ref=%d\n", rec[4 * i], rec[4 * i + 1], (int)rec[4 * i + 2], (int)rec[4 * i + 3]);
    unsigned z = 0;
    cudaMemcpyToSymbol(g_nrec, &z, 4);
    total_bad += *bad;
    total_pairs += *pairs;
  }
  printf("mismatches %llu pairs %llu err %s\n", total_bad, total_pairs, cudaGetErrorString(cudaGetLastError()));
  return total_bad == 0 ? 0 : 1;
}
