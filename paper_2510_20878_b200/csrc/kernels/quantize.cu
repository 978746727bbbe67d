// a3 + a4 of the HA-RAG hot path on sm_100a: per-group statistics and
// encode + bit-pack of one item's (layer, head) slabs into the packed blob of
// DESIGN.md §4.  Compress-once (Alg. 1 step 3); schemes:
//   INT8   P:144, symmetric absmax per group of G (R1-R3)
//   INT4   north_star, min-max per group, two codes per byte (R4)
//   FP8    P:144, E4M3 / E5M2 RNE saturating (R5) via cvt.rn.satfinite
//   GSE-8  P:155-172: per-slab exponent range -> shared-exponent array
//          ("rule C", R6), then the three steps of P:157-161 (truncation, R9)
//   PASS16 source bits unchanged
// Every fp decision is one IEEE fp32 operation with round-to-nearest-even
// (__fdiv_rn, __fsub_rn, __fadd_rn; no reciprocal, no contraction, R3).
//
// Work decomposition: a warp owns a 256-element chunk (8 elements = one
// 16-byte load per lane) of one slab and grid-strides over the item.  For
// G <= 256 a group is G/8 consecutive lanes and its statistics are a segmented
// warp-shuffle reduction — one read of the source, one write of codes + meta.
// G > 256 (e.g. the paper-ratio mode G = T*D): one warp per group, two passes
// (the second read hits L2).  GSE-8 needs the slab-wide exponent range first:
// a reduction kernel (warp shuffles + one atomicMin/Max per warp) then the
// encode kernel, which rebuilds the shared-exponent array per warp.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"

#include <unordered_map>

namespace harag {
namespace {

constexpr int kQThreads = 256;
constexpr int kChunk = 256;  // elements per warp iteration

template <int DT>
__device__ __forceinline__ float to_f32(uint32_t bits16) {
  if constexpr (DT == HR_BF16) {
    return __uint_as_float(bits16 << 16);
  } else {
    return __half2float(__ushort_as_half((unsigned short)bits16));
  }
}

// 8 source elements (one 16-byte vector) -> fp32
template <int DT>
__device__ __forceinline__ void load8(const uint16_t* p, float (&x)[8], uint4& raw) {
  raw = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[2 * i] = to_f32<DT>(w[i] & 0xFFFFu);
    x[2 * i + 1] = to_f32<DT>(w[i] >> 16);
  }
}

__device__ __forceinline__ bool any_nonfinite(const float (&x)[8]) {
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) bad |= !isfinite(x[i]);
  return bad;
}

// rne(fl(x / s)) for 8 elements of one group — the quantised codes of R3 — without an IEEE
// division per element.  y = rcp.approx(s) has relative error <= 2^-23, so t = RN(x*y) is within
// |x/s| * 1.5 * 2^-23 <= 1.5 * 2^-16 of x/s (|x/s| <= 128), and fl(x/s) within 2^-18 of x/s:
// unless t lies within 2^-15 of a half-integer, x/s, fl(x/s) and t round to the same integer.
// Elements near a half-integer (or any element when s / y are not normal) use __fdiv_rn.
__device__ __forceinline__ void div_rne8(const float (&x)[8], float s, int (&q)[8]) {
  float y;
  asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(s));
  const bool slow = !(s >= 1.17549435e-38f && s <= 8.50705917e+37f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float t = __fmul_rn(x[i], y);
    float r = rintf(t);
    // bf16 data makes exact half-integer quotients common (~0.2% of elements): only the flagged
    // element takes the IEEE division
    if (slow || fabsf(fabsf(__fsub_rn(t, r)) - 0.5f) <= 3.0517578125e-05f) r = rintf(__fdiv_rn(x[i], s));
    q[i] = (int)r;
  }
}

// sub(a, b) of R4: fl(a - b) saturated at FLT_MAX (finite inputs whose difference overflows)
__device__ __forceinline__ float sub_sat(float a, float b) { return fminf(__fsub_rn(a, b), 3.40282347e+38f); }

// segmented reductions over `seg` consecutive lanes (seg a power of two <= 32)
__device__ __forceinline__ float seg_max(float v, int seg) {
  for (int o = seg >> 1; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ float seg_min(float v, int seg) {
  for (int o = seg >> 1; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

struct Geo {  // slab addressing shared by the kernels
  const uint16_t* src;
  uint8_t* codes;
  uint8_t* meta;
};
__device__ __forceinline__ Geo slab_geo(const QuantParams& p, uint32_t slab_i) {
  const uint32_t l = slab_i / p.Hl, hl = slab_i - l * p.Hl;
  const uint64_t slab = (uint64_t)p.T * p.D;
  return {p.src + ((uint64_t)l * p.H + p.h0 + hl) * slab, p.dst + slab_i * p.code_bytes_slab,
          p.dst + p.meta_offset + slab_i * p.meta_stride};
}

// Blocked distribution: warp w of the grid owns chunks [n*w/W, n*(w+1)/W) and walks them in
// order, advancing (slab, offset) without divisions; the next chunk's load is issued before the
// current chunk is encoded (two 16-byte loads in flight per lane).
struct Walker {
  uint32_t c, c1, slab_i, e0, cps;
  Geo g;
  __device__ __forceinline__ void init(const QuantParams& p) {
    const uint32_t n = p.L * p.Hl * (p.T * p.D / kChunk);
    const uint32_t warps = gridDim.x * (kQThreads / 32);
    const uint32_t w = blockIdx.x * (kQThreads / 32) + threadIdx.x / 32;
    cps = p.T * p.D / kChunk;
    c = (uint32_t)((uint64_t)n * w / warps);
    c1 = (uint32_t)((uint64_t)n * (w + 1) / warps);
    slab_i = c / cps;
    e0 = (c - slab_i * cps) * kChunk;
    g = slab_geo(p, slab_i);
  }
  __device__ __forceinline__ bool more() const { return c < c1; }
  __device__ __forceinline__ void next(const QuantParams& p) {
    ++c;
    e0 += kChunk;
    if (e0 == cps * kChunk && c < c1) {
      e0 = 0;
      g = slab_geo(p, ++slab_i);
    }
  }
};

// ---------------------------------------------------------------- INT8 / INT4 (G <= 256)
// fl(a / 127) for the INT8 scale without a division: q0 = RN(a * y), y = RN(1/127); the residual
// r = a - 127*q0 is exact (one FMA) and RN(q0 + r*y) is the correctly rounded quotient (Markstein's
// correction).  a is always a 16-bit source value, so the identity is checked against __fdiv_rn for
// every finite bf16 and fp16 magnitude by tests/test_gpu_parity.py::test_int8_scale_all_16bit_values;
// tiny a (below 2^-100) takes the IEEE division.
__device__ __forceinline__ float div127(float a) {
  constexpr float y = 0.007874015718698501587f;  // RN(1/127)
  if (a < 7.8886090522101181e-31f) return __fdiv_rn(a, 127.f);
  const float q0 = __fmul_rn(a, y);
  const float r = __fmaf_rn(-q0, 127.f, a);
  return __fmaf_rn(r, y, q0);
}

template <int SEG>
__device__ __forceinline__ uint32_t seg_max_u32(uint32_t v) {
#pragma unroll
  for (int o = SEG >> 1; o; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
template <int SEG>
__device__ __forceinline__ float seg_min_f(float v) {
#pragma unroll
  for (int o = SEG >> 1; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
template <int SEG>
__device__ __forceinline__ float seg_max_f(float v) {
#pragma unroll
  for (int o = SEG >> 1; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// largest |x| bit pattern of the 8 16-bit values (magnitude order == integer order, NaN/Inf on top)
__device__ __forceinline__ uint32_t absmax_bits(const uint4& raw) {
  const uint32_t m = 0x7FFF7FFFu;
  const uint32_t v = __vmaxu2(__vmaxu2(raw.x & m, raw.y & m), __vmaxu2(raw.z & m, raw.w & m));
  return max(v & 0xFFFFu, v >> 16);
}

template <int SCHEME, int SEG, int DT>
__device__ __forceinline__ void encode_group_chunk(const QuantParams& p, const Geo& g, uint32_t e, const float (&x)[8],
                                                   const uint4& raw, uint32_t lane, bool& bad) {
  const uint32_t grp = e >> p.g_shift;
  const bool leader = (lane & (SEG - 1)) == 0;
  int q[8];
  if constexpr (SCHEME == HR_S_INT8) {
    // a3: a = max |x| (exact: the largest magnitude bit pattern); s = 1 if a == 0 else fl(a / 127)
    const uint32_t ab = seg_max_u32<SEG>(absmax_bits(raw));
    bad |= ab >= (DT == HR_BF16 ? 0x7F80u : 0x7C00u);  // NaN/Inf in the group
    const float a = to_f32<DT>(ab);
    const float s = (a == 0.f) ? 1.f : div127(a);
    if (leader) reinterpret_cast<float*>(g.meta)[grp] = s;
    // a4: q = clamp(rne(fl(x / s)), -127, 127).  fl(x/s) by Markstein's correction with y = RN(1/s):
    // equal to IEEE division for every (a, x) pair of 16-bit values when s is in [2^-90, 2^125]
    // (tests/csrc/markstein_check.cu, exhaustive); outside that range the IEEE division.  |x| <= a
    // gives |x/s| <= 127 (1 + 2^-24), so the clamp never binds and is omitted.
    const bool fast = s >= 8.0779356e-28f && s <= 4.2535296e+37f;
    int c8[8];
    if (__all_sync(0xFFFFFFFFu, fast)) {  // warp-uniform: the branch-free path for every normal scale
      const float y = __fdiv_rn(1.f, s);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float q0 = __fmul_rn(x[i], y);
        c8[i] = __float2int_rn(__fmaf_rn(__fmaf_rn(-q0, s, x[i]), y, q0));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) c8[i] = __float2int_rn(__fdiv_rn(x[i], s));
    }
    const uint32_t w0 = __byte_perm(__byte_perm(c8[0], c8[1], 0x0040), __byte_perm(c8[2], c8[3], 0x0040), 0x5410);
    const uint32_t w1 = __byte_perm(__byte_perm(c8[4], c8[5], 0x0040), __byte_perm(c8[6], c8[7], 0x0040), 0x5410);
    *reinterpret_cast<uint2*>(g.codes + e) = make_uint2(w0, w1);
  } else {
    bad |= any_nonfinite(x);
    // a3: mn = min + 0, mx = max + 0 (a zero extreme is +0); s = (mx == mn) ? 1 : fl(sub(mx, mn) / 15)
    float mn = x[0], mx = x[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) mn = fminf(mn, x[i]), mx = fmaxf(mx, x[i]);
    mn = __fadd_rn(seg_min_f<SEG>(mn), 0.f);
    mx = __fadd_rn(seg_max_f<SEG>(mx), 0.f);
    const float s = (mx == mn) ? 1.f : __fdiv_rn(sub_sat(mx, mn), 15.f);
    if (leader) reinterpret_cast<float2*>(g.meta)[grp] = make_float2(s, mn);
    // a4: q = clamp(rne(fl(sub(x, mn) / s)), 0, 15); element 2i -> low nibble (R24)
    float u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = sub_sat(x[i], mn);
    div_rne8(u, s, q);
    uint32_t w = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint32_t)max(0, min(15, q[i])) << (4 * i);
    *reinterpret_cast<uint32_t*>(g.codes + e / 2) = w;
  }
}

template <int SCHEME, int SEG, int DT>
__global__ void __launch_bounds__(kQThreads) quant_group_kernel(QuantParams p) {
  constexpr int kBatch = 4;  // chunks whose loads are in flight together (4 x 16 B per lane)
  const uint32_t lane = threadIdx.x & 31;
  Walker wk;
  wk.init(p);
  bool bad = false;
  while (wk.more()) {
    uint4 raw[kBatch];
    Geo g[kBatch];
    uint32_t e[kBatch];
    int n = 0;
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (wk.more()) {  // warp-uniform
        g[b] = wk.g;
        e[b] = wk.e0 + lane * 8;
        raw[b] = __ldg(reinterpret_cast<const uint4*>(wk.g.src + e[b]));
        wk.next(p);
        n = b + 1;
      }
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (b < n) {
        float x[8];
        const uint32_t w[4] = {raw[b].x, raw[b].y, raw[b].z, raw[b].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) x[2 * i] = to_f32<DT>(w[i] & 0xFFFFu), x[2 * i + 1] = to_f32<DT>(w[i] >> 16);
        encode_group_chunk<SCHEME, SEG, DT>(p, g[b], e[b], x, raw[b], lane, bad);
      }
    }
  }
  if (bad) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------- INT8 / INT4 (G > 256): warp per group
template <int SCHEME, int DT>
__global__ void __launch_bounds__(kQThreads) quant_biggroup_kernel(QuantParams p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t slab = (uint64_t)p.T * p.D;
  const uint32_t groups_per_slab = (uint32_t)(slab / p.G);
  const uint64_t n_groups = (uint64_t)p.L * p.Hl * groups_per_slab;
  bool bad = false;
  for (uint64_t gi = (blockIdx.x * (uint64_t)kQThreads + threadIdx.x) / 32; gi < n_groups;
       gi += (uint64_t)gridDim.x * kQThreads / 32) {
    const uint32_t slab_i = (uint32_t)(gi / groups_per_slab);
    const uint32_t grp = (uint32_t)(gi - (uint64_t)slab_i * groups_per_slab);
    const Geo g = slab_geo(p, slab_i);
    const uint32_t base = grp * p.G;
    float a = 0.f, mn = INFINITY, mx = -INFINITY;
    for (uint32_t e = base + lane * 8; e < base + p.G; e += kChunk) {  // pass 1: statistics
      float x[8];
      uint4 raw;
      load8<DT>(g.src + e, x, raw);
      bad |= any_nonfinite(x);
#pragma unroll
      for (int i = 0; i < 8; ++i) a = fmaxf(a, fabsf(x[i])), mn = fminf(mn, x[i]), mx = fmaxf(mx, x[i]);
    }
    float s, m0 = 0.f;
    if constexpr (SCHEME == HR_S_INT8) {
      a = seg_max(a, 32);
      s = (a == 0.f) ? 1.f : div127(a);
      if (lane == 0) reinterpret_cast<float*>(g.meta)[grp] = s;
    } else {
      mn = __fadd_rn(seg_min(mn, 32), 0.f);
      mx = __fadd_rn(seg_max(mx, 32), 0.f);
      s = (mx == mn) ? 1.f : __fdiv_rn(sub_sat(mx, mn), 15.f);
      m0 = mn;
      if (lane == 0) reinterpret_cast<float2*>(g.meta)[grp] = make_float2(s, mn);
    }
    for (uint32_t e = base + lane * 8; e < base + p.G; e += kChunk) {  // pass 2: encode (L2 re-read)
      float x[8];
      uint4 raw;
      load8<DT>(g.src + e, x, raw);
      int q[8];
      if constexpr (SCHEME == HR_S_INT8) {
        div_rne8(x, s, q);
        uint32_t w[2] = {0u, 0u};
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i >> 2] |= ((uint32_t)max(-127, min(127, q[i])) & 0xFFu) << (8 * (i & 3));
        *reinterpret_cast<uint2*>(g.codes + e) = make_uint2(w[0], w[1]);
      } else {
        float u[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) u[i] = sub_sat(x[i], m0);
        div_rne8(u, s, q);
        uint32_t w = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) w |= (uint32_t)max(0, min(15, q[i])) << (4 * i);
        *reinterpret_cast<uint32_t*>(g.codes + e / 2) = w;
      }
    }
  }
  if (bad) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------- FP8 / PASS16: elementwise
template <int SCHEME, int DT>
__global__ void __launch_bounds__(kQThreads) quant_elementwise_kernel(QuantParams p) {
  const uint32_t lane = threadIdx.x & 31;
  Walker wk;
  wk.init(p);
  bool bad = false;
  for (; wk.more(); wk.next(p)) {
    const uint32_t e = wk.e0 + lane * 8;
    float x[8];
    uint4 raw;
    load8<DT>(wk.g.src + e, x, raw);
    bad |= any_nonfinite(x);
    if constexpr (SCHEME == HR_S_PASS16) {
      *reinterpret_cast<uint4*>(wk.g.codes + 2ull * e) = raw;
    } else {
      constexpr __nv_fp8_interpretation_t kInterp = SCHEME == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
      uint32_t w[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {  // nearest code, ties to even, saturating (R5)
        const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(x[4 * i], x[4 * i + 1]), __NV_SATFINITE, kInterp);
        const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(x[4 * i + 2], x[4 * i + 3]), __NV_SATFINITE, kInterp);
        w[i] = (lo & 0xFFFFu) | (hi << 16);
      }
      *reinterpret_cast<uint2*>(wk.g.codes + e) = make_uint2(w[0], w[1]);
    }
  }
  if (bad) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------- GSE-8
// pass A: per-slab min/max biased exponent over nonzero normal values (R8, R9)
template <int DT>
__global__ void __launch_bounds__(kQThreads) gse_range_kernel(QuantParams p) {
  const uint32_t lane = threadIdx.x & 31;
  Walker wk;
  wk.init(p);
  const bool any_chunk = wk.more();
  bool bad = false;
  int emin = 255, emax = 0;
  uint32_t cur = wk.slab_i;
  auto flush = [&](uint32_t slab_i) {  // warp-reduce and publish the running range of one slab
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
    }
    if (lane == 0 && emax != 0) {  // stored as (255 - min, max) so a zero fill initialises it
      atomicMax(&p.gse_range[2 * slab_i], 255 - emin);
      atomicMax(&p.gse_range[2 * slab_i + 1], emax);
    }
    emin = 255, emax = 0;
  };
  for (; wk.more(); wk.next(p)) {
    if (wk.slab_i != cur) flush(cur), cur = wk.slab_i;
    float x[8];
    uint4 raw;
    load8<DT>(wk.g.src + wk.e0 + lane * 8, x, raw);
    bad |= any_nonfinite(x);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ef = (__float_as_uint(x[i]) >> 23) & 0xFF;
      if (ef != 0) emin = min(emin, ef), emax = max(emax, ef);
    }
  }
  if (any_chunk) flush(cur);
  if (bad) atomicOr(p.err, 1);
}

// pass B: shared-exponent array from the range (R6) and the three steps of P:157-161
template <int DT, int M>
__global__ void __launch_bounds__(kQThreads) gse_encode_kernel(QuantParams p) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr int step = M - 1, m = M, nmax = 1 << (7 - M);  // compile-time step: no integer division
  Walker wk;
  wk.init(p);
  uint32_t cur = 0xFFFFFFFFu;
  int lo = 0, n = 0, Emax = 0;
  for (; wk.more(); wk.next(p)) {
    const Geo& g = wk.g;
    const uint32_t e = wk.e0 + lane * 8;
    if (wk.slab_i != cur) {
      cur = wk.slab_i;
      const int rmin = 255 - p.gse_range[2 * cur], rmax = p.gse_range[2 * cur + 1];
      const bool any = rmax != 0;
      const int Emin = rmin - 127;
      Emax = rmax - 127;
      // lo = max(Emin, Emax - (2^e - 1) * step); G_i = min(lo + i*step, Emax), i < n
      lo = max(Emin, Emax - (nmax - 1) * step);
      n = any ? (Emax - lo + step - 1) / step + 1 : 0;
    }
    if (wk.e0 == 0) {
      // meta record: int8 array [2^e] (unused -128), zero pad to 16 B, then the fp32 decode table
      // [2^(e+1)]: entry (sign << e | i) = (-1)^sign 2^(G_i - (m-1)), 0 for unused i
      if (lane < 16) {
        int v = 0;
        if ((int)lane < nmax) v = ((int)lane < n) ? min(lo + (int)lane * step, Emax) : -128;
        g.meta[lane] = (uint8_t)(int8_t)v;
      }
      for (uint32_t w = lane; w < (p.meta_stride - 16) / 4; w += 32) {
        float v = 0.f;
        const int i = (int)w & (nmax - 1);
        if ((int)w < 2 * nmax && i < n) {
          const int k = min(lo + i * step, Emax) - step;
          v = k >= -126 ? __int_as_float((k + 127) << 23) : (k >= -149 ? __int_as_float(1 << (k + 149)) : 0.f);
          if ((int)w >= nmax) v = -v;
        }
        reinterpret_cast<float*>(g.meta + 16)[w] = v;
      }
    }
    float x[8];
    uint4 raw;
    load8<DT>(g.src + e, x, raw);
    uint32_t w[2] = {0u, 0u};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t b = __float_as_uint(x[i]);
      const int ef = (b >> 23) & 0xFF;
      uint32_t byte = 0u;
      if (ef != 0) {
        const int E = ef - 127;
        const int idx = (E <= lo) ? 0 : (E - lo + step - 1) / step;  // smallest G_i >= E
        const int G = min(lo + idx * step, Emax);
        const int d = G - E;
        if (d <= m - 1) {  // else below the array's reach: flush (R9)
          const int keep = m - 1 - d;
          // marker 1 at position d+1 from the MSB, then the top fraction bits (truncated)
          const uint32_t field = (1u << keep) | ((b & 0x7FFFFFu) >> (23 - keep));
          byte = ((b >> 31) << 7) | ((uint32_t)idx << m) | field;
        }
      }
      w[i >> 2] |= byte << (8 * (i & 3));
    }
    *reinterpret_cast<uint2*>(g.codes + e) = make_uint2(w[0], w[1]);
  }
}

int g_num_sms = 0;
// One wave of resident CTAs (the warps walk contiguous chunk blocks): SMs x occupancy of `kernel`.
template <class K>
int grid_for(K kernel, uint64_t warps) {
  if (!g_num_sms) {
    int dev = 0;
    HR_CUDA(cudaGetDevice(&dev));
    HR_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  static std::unordered_map<const void*, int> cache;  // occupancy per kernel
  auto it = cache.find((const void*)kernel);
  if (it == cache.end()) {
    int o = 0;
    HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, kQThreads, 0));
    it = cache.emplace((const void*)kernel, o).first;
  }
  const int occ = it->second;
  const uint64_t want = (warps * 32 + kQThreads - 1) / kQThreads;
  const uint64_t cap = (uint64_t)g_num_sms * (occ > 0 ? occ : 1);
  return (int)(want < cap ? (want ? want : 1) : cap);
}

template <int DT>
void launch_dt(const QuantParams& p, cudaStream_t st) {
  const uint64_t slab = (uint64_t)p.T * p.D;
  const uint64_t chunks = (uint64_t)p.L * p.Hl * (slab / kChunk);
#define LAUNCH(KERNEL, WORK) KERNEL<<<grid_for(KERNEL, WORK), kQThreads, 0, st>>>(p)
  switch (p.scheme) {
    case HR_S_PASS16:
      LAUNCH((quant_elementwise_kernel<HR_S_PASS16, DT>), chunks);
      break;
    case HR_S_FP8E4M3:
      LAUNCH((quant_elementwise_kernel<HR_S_FP8E4M3, DT>), chunks);
      break;
    case HR_S_FP8E5M2:
      LAUNCH((quant_elementwise_kernel<HR_S_FP8E5M2, DT>), chunks);
      break;
    case HR_S_INT8:
    case HR_S_INT4: {
      if (p.G <= (uint32_t)kChunk) {
        switch ((p.G >> 3) * 16 + (p.scheme == HR_S_INT8 ? 0 : 1)) {
#define QG(SEGV)                                                        \
  case SEGV * 16 + 0: LAUNCH((quant_group_kernel<HR_S_INT8, SEGV, DT>), chunks); break; \
  case SEGV * 16 + 1: LAUNCH((quant_group_kernel<HR_S_INT4, SEGV, DT>), chunks); break;
          QG(4) QG(8) QG(16) QG(32)
#undef QG
          default: fail(HR_EINVAL, "group size must be a power of two >= 32");
        }
      } else {
        const uint64_t groups = (uint64_t)p.L * p.Hl * (slab / p.G);
        if (p.scheme == HR_S_INT8)
          LAUNCH((quant_biggroup_kernel<HR_S_INT8, DT>), groups);
        else
          LAUNCH((quant_biggroup_kernel<HR_S_INT4, DT>), groups);
      }
      break;
    }
    case HR_S_GSE8: {
      const uint64_t n_slabs = (uint64_t)p.L * p.Hl;
      HR_CUDA(cudaMemsetAsync(p.gse_range, 0, sizeof(int) * 2 * n_slabs, st));
      LAUNCH((gse_range_kernel<DT>), chunks);
      if (p.gse_m == 3)
        LAUNCH((gse_encode_kernel<DT, 3>), chunks);
      else if (p.gse_m == 4)
        LAUNCH((gse_encode_kernel<DT, 4>), chunks);
      else
        LAUNCH((gse_encode_kernel<DT, 5>), chunks);
      break;
    }
    default:
      fail(HR_EINVAL, "unknown scheme");
  }
#undef LAUNCH
  HR_CUDA(cudaGetLastError());
}

}  // namespace

void launch_quantize(const QuantParams& p, cudaStream_t st) {
  require(((uint64_t)p.T * p.D) % kChunk == 0, HR_EINVAL, "T*D must be a multiple of 256");
  if (p.dtype == HR_BF16)
    launch_dt<HR_BF16>(p, st);
  else
    launch_dt<HR_FP16>(p, st);
}

}  // namespace harag
