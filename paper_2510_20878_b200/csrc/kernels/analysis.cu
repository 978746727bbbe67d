// Analysis kernels: exponent histograms of 16-bit KV
// values (Fig. KV-exponent-range) and the compression error of
// Eq., RMSE = sqrt(1/N sum (x_i - x^_i)^2).  HBM-bound streaming
// reductions: 16-byte loads, grid of SMs x resident CTAs, one pass.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../common.h"
#include "../analysis.h"

namespace harag {

namespace {

constexpr int kHistThreads = 256;
constexpr int kHistWarps = kHistThreads / 32;
constexpr int kHistBatch = 16;       // 16-byte loads in flight per lane (256 B: 64 KB per SM)
constexpr uint32_t kFlushVecs = 8000;  // 16-bit lane counters: flush before 65535 (8 elements per vector)

// Biased exponent field of a 16-bit float: bf16 bits 14..7 (8 bits), fp16 bits 14..10 (5 bits).
template <int DT>
__device__ __forceinline__ uint32_t exp_field(uint32_t bits16) {
  return DT == HR_BF16 ? (bits16 >> 7) & 0xFFu : (bits16 >> 10) & 0x1Fu;
}

// Lane-private 16-bit counters, two bins per word: word w = bin / 2 of lane L lives at
// cnt[w * 32 + (L ^ (w & 31))] — no inter-lane conflicts (each lane owns its column) and, because
// the column is XOR-swizzled by the row, lanes counting the same bin hit 32 different banks.  The
// increment is a shared-memory reduction (no return value), so consecutive values of one lane that
// land in the same bin do not form a load -> add -> store dependency chain.
__device__ __forceinline__ void hist_add(uint32_t* cnt, uint32_t lane, uint32_t bin) {
  const uint32_t w = bin >> 1;
  atomicAdd(&cnt[w * 32 + (lane ^ (w & 31))], 1u << ((bin & 1) * 16));
}

// Sum the warp's lane counters into the block histogram and clear them: lane i reads rows i,
// i + 32, ..., with the same swizzle (conflict-free: row i, column j sits in bank j ^ i).
__device__ __forceinline__ void hist_flush(uint32_t* cnt, uint32_t lane, uint32_t* block_hist) {
  for (uint32_t w = lane; w < 128; w += 32) {
    uint32_t lo = 0, hi = 0;
#pragma unroll 8
    for (uint32_t j = 0; j < 32; ++j) {
      uint32_t& c = cnt[w * 32 + (j ^ (w & 31))];
      lo += c & 0xFFFFu, hi += c >> 16;
      c = 0;
    }
    if (lo) atomicAdd(block_hist + 2 * w, lo);
    if (hi) atomicAdd(block_hist + 2 * w + 1, hi);
  }
}

template <int DT>
__global__ void __launch_bounds__(kHistThreads) exponent_hist_kernel(const uint4* __restrict__ src, uint64_t n_vec,
                                                                     const uint16_t* __restrict__ tail,
                                                                     uint32_t n_tail,
                                                                     unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t hsm[];  // [warps][128 words][32 lanes] + block histogram [256]
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* cnt = hsm + warp * 128 * 32;
  uint32_t* bh = hsm + kHistWarps * 128 * 32;
  for (uint32_t i = threadIdx.x; i < kHistWarps * 128 * 32 + 256; i += kHistThreads) hsm[i] = 0;
  __syncthreads();
  // blocked distribution: warp gw owns vectors [n*gw/W, n*(gw+1)/W), walked 32 lanes x 8 at a time
  const uint64_t W = (uint64_t)gridDim.x * kHistWarps, gw = (uint64_t)blockIdx.x * kHistWarps + warp;
  const uint64_t v0 = n_vec * gw / W, v1 = n_vec * (gw + 1) / W;
  uint32_t since = 0;
  for (uint64_t vb = v0; vb < v1; vb += 32 * kHistBatch) {  // warp-uniform trip count
    const uint64_t v = vb + lane;
    uint4 q[kHistBatch];
#pragma unroll
    for (int b = 0; b < kHistBatch; ++b)
      if (v + 32ull * b < v1) q[b] = __ldcs(src + v + 32ull * b);
#pragma unroll
    for (int b = 0; b < kHistBatch; ++b) {
      if (v + 32ull * b < v1) {
        const uint32_t w[4] = {q[b].x, q[b].y, q[b].z, q[b].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          hist_add(cnt, lane, exp_field<DT>(w[j] & 0xFFFFu));
          hist_add(cnt, lane, exp_field<DT>(w[j] >> 16));
        }
      }
    }
    since += kHistBatch;
    if (since >= kFlushVecs) {  // warp-uniform (every lane runs the same number of iterations)
      __syncwarp();
      hist_flush(cnt, lane, bh);
      __syncwarp();
      since = 0;
    }
  }
  if (blockIdx.x == 0 && warp == 0)
    for (uint32_t i = lane; i < n_tail; i += 32) hist_add(cnt, lane, exp_field<DT>(tail[i]));
  __syncwarp();
  hist_flush(cnt, lane, bh);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < 256; b += kHistThreads)
    if (bh[b]) atomicAdd(hist + b, (unsigned long long)bh[b]);
}

__device__ __forceinline__ float to_f32(uint32_t bits16, uint32_t dt) {
  return dt == HR_BF16 ? __uint_as_float(bits16 << 16) : __half2float(__ushort_as_half((unsigned short)bits16));
}

constexpr int kErrThreads = 256;

// Per-block partial sum of squared differences (fp64) and max |difference| between this
// rank's heads of a source item x ([L][H][T][D]) and a decoded item y ([L][Hl][T][D]).
__global__ void __launch_bounds__(kErrThreads) error_partial_kernel(const uint16_t* __restrict__ x,
                                                                    const uint16_t* __restrict__ y, uint32_t L,
                                                                    uint32_t H, uint32_t Hl, uint32_t h0,
                                                                    uint64_t slab, uint32_t dt,
                                                                    double* __restrict__ part_sse,
                                                                    double* __restrict__ part_max) {
  const uint64_t slab_v = slab / 8;  // 16-byte vectors per slab (slab % 256 == 0)
  const uint64_t n_vec = (uint64_t)L * Hl * slab_v;
  double sse = 0.0, mx = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kErrThreads;
  for (uint64_t v = (uint64_t)blockIdx.x * kErrThreads + threadIdx.x; v < n_vec; v += stride) {
    const uint64_t s = v / slab_v, off = v - s * slab_v;
    const uint64_t l = s / Hl, hh = s - l * Hl;
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(x + ((l * H + h0 + hh) * slab)) + off);
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(y) + v);
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t sh = (j & 1) * 16;
      // both values are exact in fp32; their difference is exact in fp64
      const double d = (double)to_f32((wa[j >> 1] >> sh) & 0xFFFFu, dt) - (double)to_f32((wb[j >> 1] >> sh) & 0xFFFFu, dt);
      sse = fma(d, d, sse);
      mx = fmax(mx, fabs(d));
    }
  }
  __shared__ double ss[kErrThreads], sm[kErrThreads];
  ss[threadIdx.x] = sse;
  sm[threadIdx.x] = mx;
  __syncthreads();
  for (int w = kErrThreads / 2; w > 0; w >>= 1) {  // fixed tree: deterministic run to run
    if (threadIdx.x < w) {
      ss[threadIdx.x] += ss[threadIdx.x + w];
      sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part_sse[blockIdx.x] = ss[0], part_max[blockIdx.x] = sm[0];
}

__global__ void error_final_kernel(const double* __restrict__ part_sse, const double* __restrict__ part_max,
                                   uint32_t n, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, m = 0.0;
  for (uint32_t i = 0; i < n; ++i) s += part_sse[i], m = fmax(m, part_max[i]);  // fixed order
  out[0] = s, out[1] = m;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Value-distribution guard (R29): one CTA per (layer, head) slab of an item's source
// [L][H][slab] (ALL heads).  Pass 1: min / max fp32 exponent field over the nonzero normals and max |x|;
// rule C's first shared exponent lo = max(Emin, Emax - (2^e - 1)(m - 1)) (R6); pass 2 (the slab again,
// from L1/L2) counts the nonzero values GSE-8 flushes to field 0: fp32 subnormals and E < lo - (m - 1)
// (R9).  stats[0] += the count, stats[1] = max(stats[1], bits of max |x|) (non-negative fp32 bits order
// like the values).
constexpr int kGuardThreads = 256;
template <int DT>
__device__ __forceinline__ uint32_t f32_bits(uint32_t bits16) {
  return DT == HR_BF16 ? bits16 << 16 : __float_as_uint(__half2float(__ushort_as_half((unsigned short)bits16)));
}
template <int DT>
__global__ void __launch_bounds__(kGuardThreads) guard_kernel(const uint16_t* __restrict__ src, uint32_t slab,
                                                              int e_bits, int m_bits,
                                                              unsigned long long* __restrict__ stats) {
  __shared__ uint32_t red[3][kGuardThreads / 32];
  __shared__ uint32_t thr_s;
  const uint4* v = reinterpret_cast<const uint4*>(src + (uint64_t)blockIdx.x * slab);
  const uint32_t nv = slab / 8, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t emin = 255, emax = 0, amax = 0;
  for (uint32_t i = threadIdx.x; i < nv; i += kGuardThreads) {
    const uint4 w = __ldg(v + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t b = f32_bits<DT>((ws[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) & 0x7FFFFFFFu;
      const uint32_t ef = b >> 23;
      amax = max(amax, b);
      if (ef != 0) emin = min(emin, ef), emax = max(emax, ef);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
    emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
    amax = max(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, o));
  }
  if (lane == 0) red[0][warp] = emin, red[1][warp] = emax, red[2][warp] = amax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kGuardThreads / 32; ++w)
      emin = min(emin, red[0][w]), emax = max(emax, red[1][w]), amax = max(amax, red[2][w]);
    // biased threshold: fields below it (and every nonzero subnormal) flush; no normal value at all ->
    // every nonzero value flushes
    int thr = 256;
    if (emax != 0) {
      const int step = m_bits - 1;
      const int lo = max((int)emin - 127, (int)emax - 127 - ((1 << e_bits) - 1) * step);
      thr = lo - step + 127;
    }
    thr_s = (uint32_t)max(thr, 1);
    atomicMax(stats + 1, (unsigned long long)amax);
  }
  __syncthreads();
  const uint32_t thr = thr_s;
  uint32_t cnt = 0;
  for (uint32_t i = threadIdx.x; i < nv; i += kGuardThreads) {
    const uint4 w = __ldg(v + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t b = f32_bits<DT>((ws[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) & 0x7FFFFFFFu;
      cnt += (b != 0u && (b >> 23) < thr) ? 1u : 0u;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(stats, (unsigned long long)cnt);
}

}  // namespace

void launch_guard(uint32_t dtype, const void* src, uint64_t n_slabs, uint64_t slab, uint32_t e_bits,
                  uint32_t m_bits, unsigned long long* stats, cudaStream_t st) {
  require(slab % 8 == 0 && slab < (1ull << 32), HR_EINVAL, "guard: slab must be a multiple of 8 elements");
  require(reinterpret_cast<uintptr_t>(src) % 16 == 0, HR_EINVAL, "guard: source must be 16-byte aligned");
  require(n_slabs < (1ull << 31), HR_EINVAL, "guard: too many slabs");
  if (!n_slabs) return;
  if (dtype == HR_BF16)
    guard_kernel<HR_BF16><<<(unsigned)n_slabs, kGuardThreads, 0, st>>>(static_cast<const uint16_t*>(src),
                                                                       (uint32_t)slab, (int)e_bits, (int)m_bits, stats);
  else
    guard_kernel<HR_FP16><<<(unsigned)n_slabs, kGuardThreads, 0, st>>>(static_cast<const uint16_t*>(src),
                                                                       (uint32_t)slab, (int)e_bits, (int)m_bits, stats);
  HR_CUDA(cudaGetLastError());
}

void launch_exponent_hist(uint32_t dtype, const void* src, uint64_t n, unsigned long long* hist,
                          cudaStream_t stream) {
  const uint64_t n_vec = (reinterpret_cast<uintptr_t>(src) % 16 == 0) ? n / 8 : 0;
  const uint64_t n_tail = n - n_vec * 8;
  require(n_tail < (1u << 20), HR_EINVAL, "source must be 16-byte aligned for large inputs");
  const uint16_t* tail = static_cast<const uint16_t*>(src) + n_vec * 8;
  const size_t smem = (kHistWarps * 128 * 32 + 256) * sizeof(uint32_t);
  static bool init[2] = {false, false};
  auto kern = dtype == HR_BF16 ? exponent_hist_kernel<HR_BF16> : exponent_hist_kernel<HR_FP16>;
  if (!init[dtype & 1]) {
    HR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    init[dtype & 1] = true;
  }
  int occ = 0;
  HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kHistThreads, smem));
  const uint64_t want = std::max<uint64_t>(1, (n_vec + 32 * kHistBatch * kHistWarps - 1) / (32 * kHistBatch * kHistWarps));
  const int grid = (int)std::min<uint64_t>((uint64_t)std::max(1, occ) * sm_count(), want);
  kern<<<grid, kHistThreads, smem, stream>>>(static_cast<const uint4*>(src), n_vec, tail, (uint32_t)n_tail, hist);
}

uint32_t error_partials(uint64_t n_elems) {
  return (uint32_t)std::min<uint64_t>(8 * sm_count(), std::max<uint64_t>(1, n_elems / (8 * kErrThreads)));
}

void launch_error(const uint16_t* x, const uint16_t* y, uint32_t L, uint32_t H, uint32_t Hl, uint32_t h0,
                  uint64_t slab, uint32_t dtype, double* partials, uint32_t n_part, double* out,
                  cudaStream_t stream) {
  error_partial_kernel<<<n_part, kErrThreads, 0, stream>>>(x, y, L, H, Hl, h0, slab, dtype, partials,
                                                           partials + n_part);
  error_final_kernel<<<1, 32, 0, stream>>>(partials, partials + n_part, n_part, out);
}

}  // namespace harag
