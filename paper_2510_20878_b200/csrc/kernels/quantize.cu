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
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"

namespace harag {
namespace {

constexpr int kQThreads = 256;

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

__device__ __forceinline__ uint32_t ord_key(float f) {  // float order == unsigned order
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord_unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

template <int SCHEME, int DT>
__global__ void __launch_bounds__(kQThreads) quantize_slab_kernel(QuantParams p) {
  extern __shared__ __align__(16) uint32_t qsm[];
  const uint32_t slab_id = blockIdx.x;  // = l * Hl + h_local
  const uint32_t l = slab_id / p.Hl, hl = slab_id % p.Hl;
  const uint64_t slab = (uint64_t)p.T * p.D;
  const uint16_t* src = p.src + ((uint64_t)l * p.H + p.h0 + hl) * slab;
  uint8_t* codes = p.dst + slab_id * p.code_bytes_slab;
  uint8_t* meta = p.dst + p.meta_offset + slab_id * p.meta_stride;
  const uint32_t n_vec = (uint32_t)(slab / 8);
  const uint32_t ng = (uint32_t)(slab / p.G);
  const uint32_t tid = threadIdx.x;
  bool bad = false;

  if constexpr (SCHEME == HR_S_PASS16) {
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
#pragma unroll
      for (int i = 0; i < 8; ++i) bad |= !isfinite(x[i]);
      reinterpret_cast<uint4*>(codes)[v] = raw;
    }
  } else if constexpr (SCHEME == HR_S_FP8E4M3 || SCHEME == HR_S_FP8E5M2) {
    constexpr __nv_fp8_interpretation_t kInterp = SCHEME == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      uint32_t w[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(x[4 * i], x[4 * i + 1]), __NV_SATFINITE, kInterp);
        uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(x[4 * i + 2], x[4 * i + 3]), __NV_SATFINITE, kInterp);
        w[i] = (lo & 0xFFFFu) | (hi << 16);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) bad |= !isfinite(x[i]);
      reinterpret_cast<uint2*>(codes)[v] = make_uint2(w[0], w[1]);
    }
  } else if constexpr (SCHEME == HR_S_INT8) {
    uint32_t* amax = qsm;  // |x| bits per group (non-negative floats order as unsigned)
    float* scale = reinterpret_cast<float*>(qsm + ng);
    for (uint32_t g = tid; g < ng; g += kQThreads) amax[g] = 0u;
    __syncthreads();
    // a3: a = max |x| per group
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bad |= !isfinite(x[i]);
        a = fmaxf(a, fabsf(x[i]));
      }
      atomicMax(&amax[(8ull * v) / p.G], __float_as_uint(a));
    }
    __syncthreads();
    // s = 1 if a == 0 else fl(a / 127)
    const uint32_t rec_words = (uint32_t)(p.meta_stride / 4);
    for (uint32_t g = tid; g < rec_words; g += kQThreads) {
      float s = 0.f;
      if (g < ng) {
        const float a = __uint_as_float(amax[g]);
        s = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
        scale[g] = s;
      }
      reinterpret_cast<float*>(meta)[g] = s;  // padding words written as 0
    }
    __syncthreads();
    // a4: q = clamp(rne(fl(x / s)), -127, 127)
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      const float s = scale[(8ull * v) / p.G];
      uint32_t w[2] = {0u, 0u};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int q = __float2int_rn(__fdiv_rn(x[i], s));
        q = max(-127, min(127, q));
        w[i >> 2] |= ((uint32_t)q & 0xFFu) << (8 * (i & 3));
      }
      reinterpret_cast<uint2*>(codes)[v] = make_uint2(w[0], w[1]);
    }
  } else if constexpr (SCHEME == HR_S_INT4) {
    uint32_t* kmin = qsm;
    uint32_t* kmax = qsm + ng;
    float* scale = reinterpret_cast<float*>(qsm + 2 * ng);
    float* minv = reinterpret_cast<float*>(qsm + 3 * ng);
    for (uint32_t g = tid; g < ng; g += kQThreads) kmin[g] = 0xFFFFFFFFu, kmax[g] = 0u;
    __syncthreads();
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      float mn = x[0], mx = x[0];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bad |= !isfinite(x[i]);
        mn = fminf(mn, x[i]);
        mx = fmaxf(mx, x[i]);
      }
      const uint32_t g = (uint32_t)((8ull * v) / p.G);
      atomicMin(&kmin[g], ord_key(mn));
      atomicMax(&kmax[g], ord_key(mx));
    }
    __syncthreads();
    const uint32_t rec_words = (uint32_t)(p.meta_stride / 4);
    for (uint32_t w = tid; w < rec_words; w += kQThreads) {
      float val = 0.f;
      const uint32_t g = w >> 1;
      if (g < ng) {
        // mn = min + 0, mx = max + 0 (a zero extreme is +0); s = (mx == mn) ? 1 : fl(fl(mx - mn) / 15)
        const float mn = __fadd_rn(ord_unkey(kmin[g]), 0.f);
        const float mx = __fadd_rn(ord_unkey(kmax[g]), 0.f);
        const float s = (mx == mn) ? 1.f : __fdiv_rn(__fsub_rn(mx, mn), 15.f);
        if ((w & 1) == 0) scale[g] = s, minv[g] = mn;
        val = (w & 1) ? mn : s;
      }
      reinterpret_cast<float*>(meta)[w] = val;
    }
    __syncthreads();
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      const uint32_t g = (uint32_t)((8ull * v) / p.G);
      const float s = scale[g], mn = minv[g];
      uint32_t w = 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int q = __float2int_rn(__fdiv_rn(__fsub_rn(x[i], mn), s));
        q = max(0, min(15, q));
        w |= (uint32_t)q << (4 * i);  // element 2i -> low nibble (R24)
      }
      reinterpret_cast<uint32_t*>(codes)[v] = w;
    }
  } else if constexpr (SCHEME == HR_S_GSE8) {
    int* rng = reinterpret_cast<int*>(qsm);  // [0] = min biased exponent, [1] = max, [2] = lo, [3] = n
    if (tid == 0) rng[0] = 255, rng[1] = 0;
    __syncthreads();
    // a3: exponent range over nonzero normal values (R8, R9)
    int emin = 255, emax = 0;
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bad |= !isfinite(x[i]);
        const int ef = (__float_as_uint(x[i]) >> 23) & 0xFF;
        if (ef != 0) emin = min(emin, ef), emax = max(emax, ef);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
    }
    if ((tid & 31) == 0) atomicMin(&rng[0], emin), atomicMax(&rng[1], emax);
    __syncthreads();
    const int step = (int)p.gse_m - 1;
    const int nmax = 1 << p.gse_e;
    const bool any = rng[1] != 0;
    const int Emin = rng[0] - 127, Emax = rng[1] - 127;
    // P:172 / R6: lo = max(Emin, Emax - (2^e - 1) * step); G_i = min(lo + i*step, Emax)
    const int lo = max(Emin, Emax - (nmax - 1) * step);
    const int n = any ? (Emax - lo + step - 1) / step + 1 : 0;
    // meta record: int8 array [2^e] (unused -128), zero pad to 16 B, then the fp32 decode table
    // [2^(e+1)]: entry (sign << e | i) = (-1)^sign 2^(G_i - (m-1)) (0 for unused i)
    for (uint32_t w = tid; w < 16; w += kQThreads) {
      int v = 0;
      if ((int)w < nmax) v = ((int)w < n) ? min(lo + (int)w * step, Emax) : -128;
      meta[w] = (uint8_t)(int8_t)v;
    }
    for (uint32_t w = tid; w < (p.meta_stride - 16) / 4; w += kQThreads) {
      float v = 0.f;
      const int i = (int)w & (nmax - 1);
      if ((int)w < 2 * nmax && i < n) {
        const int k = min(lo + i * step, Emax) - (step);  // G_i - (m-1)
        v = k >= -126 ? __int_as_float((k + 127) << 23) : (k >= -149 ? __int_as_float(1 << (k + 149)) : 0.f);
        if ((int)w >= nmax) v = -v;
      }
      reinterpret_cast<float*>(meta + 16)[w] = v;
    }
    const int m = (int)p.gse_m;
    for (uint32_t v = tid; v < n_vec; v += kQThreads) {
      float x[8];
      uint4 raw;
      load8<DT>(src + 8ull * v, x, raw);
      uint32_t w[2] = {0u, 0u};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t b = __float_as_uint(x[i]);
        const int ef = (b >> 23) & 0xFF;
        uint32_t byte = 0u;
        if (ef != 0) {
          const int E = ef - 127;
          // smallest shared exponent >= E
          const int idx = (E <= lo) ? 0 : (E - lo + step - 1) / step;
          const int G = min(lo + idx * step, Emax);
          const int d = G - E;
          if (d <= m - 1) {  // else: below the array's reach, flush (R9)
            const int keep = m - 1 - d;
            // marker 1 at position d+1 from the MSB, then the top fraction bits (truncated)
            const uint32_t field = (1u << keep) | ((b & 0x7FFFFFu) >> (23 - keep));
            byte = ((b >> 31) << 7) | ((uint32_t)idx << m) | field;
          }
        }
        w[i >> 2] |= byte << (8 * (i & 3));
      }
      reinterpret_cast<uint2*>(codes)[v] = make_uint2(w[0], w[1]);
    }
  }
  if (bad) atomicOr(p.err, 1);
}

template <int SCHEME>
void launch_q(const QuantParams& p, cudaStream_t st) {
  const uint32_t ng = (uint32_t)((uint64_t)p.T * p.D / p.G);
  size_t smem = SCHEME == HR_S_INT8 ? 8ull * ng : SCHEME == HR_S_INT4 ? 16ull * ng : 16;
  const dim3 grid(p.L * p.Hl);
  if (smem > 48 * 1024) {
    HR_CUDA(cudaFuncSetAttribute(quantize_slab_kernel<SCHEME, HR_BF16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HR_CUDA(cudaFuncSetAttribute(quantize_slab_kernel<SCHEME, HR_FP16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  if (p.dtype == HR_BF16)
    quantize_slab_kernel<SCHEME, HR_BF16><<<grid, kQThreads, smem, st>>>(p);
  else
    quantize_slab_kernel<SCHEME, HR_FP16><<<grid, kQThreads, smem, st>>>(p);
  HR_CUDA(cudaGetLastError());
}

}  // namespace

void launch_quantize(const QuantParams& p, cudaStream_t st) {
  switch (p.scheme) {
    case HR_S_PASS16: return launch_q<HR_S_PASS16>(p, st);
    case HR_S_INT8: return launch_q<HR_S_INT8>(p, st);
    case HR_S_FP8E4M3: return launch_q<HR_S_FP8E4M3>(p, st);
    case HR_S_FP8E5M2: return launch_q<HR_S_FP8E5M2>(p, st);
    case HR_S_GSE8: return launch_q<HR_S_GSE8>(p, st);
    case HR_S_INT4: return launch_q<HR_S_INT4>(p, st);
    default: fail(HR_EINVAL, "unknown scheme");
  }
}

}  // namespace harag
