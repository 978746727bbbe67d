// a3 + a4 of the HA-RAG hot path on sm_100a: per-group statistics and
// encode + bit-pack of items' (layer, head) slabs into the packed blob of
// DESIGN.md §4.  Compress-once (Alg. 1 step 3); schemes:
//   INT8   P:144, symmetric absmax per group of G (R1-R3)
//   INT4   north_star, min-max per group, two codes per byte (R4)
//   FP8    P:144, E4M3 / E5M2 RNE saturating (R5) via cvt.rn.satfinite
//   GSE-8  P:155-172: per-slab exponent range -> shared-exponent array
//          ("rule C", R6), then the three steps of P:157-161 (truncation, R9)
//   PASS16 source bits unchanged
// Every integer-deciding fp decision equals one IEEE fp32 operation with
// round-to-nearest-even (R3); where the kernel avoids a division it proves
// equality (Markstein's correction, exhaustively checked) or falls back to
// __fdiv_rn near a rounding tie.
//
// Structure (warp-specialised, persistent, batched): one launch quantises a
// batch of items (the K and V of a doc, or more), possibly of different
// schemes.  Work unit = tile of kQRingTileE (ring) or kQTileE (tile kernel) consecutive source elements of one
// (item, layer, head) slab.  CTA = 1 producer warp + kQWarps consumer warps,
// one CTA per SM, CTA b owns a contiguous block of tiles.  The producer's lane
// 0 has the TMA engine bulk-copy each tile's 16-bit source into a kQStages-deep
// shared-memory ring (mbarrier full / empty); for GSE-8 the whole producer
// warp also builds the tile's 256-entry exponent -> code-template table from
// the slab's exponent range and writes the slab's meta record.  Consumer warps
// encode 256-element chunks straight from shared memory (segmented warp-shuffle
// group statistics for INT8 / INT4: the source is read from HBM once) and store
// codes and scales; PASS16 tiles are written back by the bulk-copy engine.
// GSE-8 needs the slab-wide exponent range before any code: a range pass
// (same kernel, RANGE mode: read-only) precedes the encode launch; for a K+V
// batch (67 MB at Llama-3-8B shape) the encode's re-read hits the 126 MB L2.
//
// Group sizes G > 256 (the "paper-ratio" mode G = T*D) use
// quant_biggroup_kernel: one warp per group, two passes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"
#include "ptx.h"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>

namespace harag {
namespace {

using namespace ptx;

#ifndef HARAG_Q_WARPS
#define HARAG_Q_WARPS 16
#endif
#ifndef HARAG_Q_STAGES
#define HARAG_Q_STAGES 3
#endif
#ifndef HARAG_Q_TILE
#define HARAG_Q_TILE 16384
#endif
#ifndef HARAG_Q_RING_TILE
#define HARAG_Q_RING_TILE 32768
#endif
constexpr int kQWarps = HARAG_Q_WARPS;           // consumer warps per CTA
constexpr int kQThreadsB = 32 * (1 + kQWarps);   // + 1 producer warp
constexpr int kQStages = HARAG_Q_STAGES;         // ring depth
constexpr uint32_t kQTileE = HARAG_Q_TILE;       // source elements per tile of quant_tile_kernel (2 B each)
// source elements per tile of the persistent ring: two 1,024-element steps per consumer warp and tile
// (independent statistics chains to overlap), 3 stages of 64 KiB (INT4 9.31 -> 8.64-8.68 us/item vs
// 16,384-element tiles x 4 stages; INT8 unchanged)
constexpr uint32_t kQRingTileE = HARAG_Q_RING_TILE;
constexpr int kQMaxJobs = 32;                    // items per launch
constexpr int kChunk = 256;                      // elements per warp step (8 per lane)
constexpr float kMagic = 12582912.f;             // 1.5 * 2^23: fl(v + kMagic) = rne(v) in the low bits, |v| < 2^22

enum { MODE_ENCODE = 0, MODE_RANGE = 1 };

struct QJob {
  const uint16_t* src;  // [L][H][T][D] all heads
  uint8_t* dst;         // item blob
  int* range;           // GSE-8: int[2 * L * Hl] (255 - min, max) biased exponents, zero-initialised
  uint32_t scheme;
  uint32_t pad;
};

struct QBatch {
  QJob jobs[kQMaxJobs];
  uint32_t n_jobs;
  uint32_t L, H, Hl, h0, T, D, G, g_shift, gse_e, gse_m, dtype;
  uint32_t slab, tile_e, tiles_per_slab;
  uint64_t n_tiles;
  uint64_t code_slab[HR_N_SCHEMES], meta_off[HR_N_SCHEMES];
  uint32_t meta_stride[HR_N_SCHEMES];
  int* err;
  // tail balancing (as assemble_kv_kernel): the last dyn_tiles tiles are claimed in chunks of dyn_chunk
  // through sched[0..1] (u64 counter; sched[2] counts producers done, the last one zeroes both); the rest
  // are split in blocks.  sched == nullptr: blocked split only.
  uint32_t* sched;
  uint64_t dyn_tiles;
  uint32_t dyn_chunk;
};

struct QHdr {
  uint8_t* codes;   // first code byte of the tile
  uint8_t* meta;    // INT8 / INT4: the tile's first group record; GSE-8: slab record
  int* range;       // RANGE mode: the slab's exponent-range pair
  uint32_t n_el;    // elements in the tile (multiple of 256)
  uint32_t scheme;
};

// Dynamic shared memory: [tile ring | GSE tables | headers | full | empty]
struct QSmem {
  uint8_t* base;
  __device__ __forceinline__ uint8_t* tile(int s) const { return base + (size_t)s * kQRingTileE * 2; }
  __device__ __forceinline__ uint32_t* gtab(int s) const {
    return reinterpret_cast<uint32_t*>(base + (size_t)kQStages * kQRingTileE * 2) + 256 * s;
  }
  __device__ __forceinline__ QHdr* hdr() const { return reinterpret_cast<QHdr*>(gtab(kQStages)); }
  __device__ __forceinline__ uint64_t* full() const { return reinterpret_cast<uint64_t*>(hdr() + kQStages); }
  __device__ __forceinline__ uint64_t* empty() const { return full() + kQStages; }
};
constexpr size_t kQSmemBytes =
    (size_t)kQStages * kQRingTileE * 2 + (size_t)kQStages * 1024 + kQStages * sizeof(QHdr) + 2 * kQStages * 8;

__device__ __forceinline__ uint32_t code_bytes(uint32_t scheme, uint32_t n_el) {
  return scheme == HR_S_PASS16 ? 2 * n_el : scheme == HR_S_INT4 ? n_el / 2 : n_el;
}

// ------------------------------------------------------------------ element helpers
template <int DT>
__device__ __forceinline__ float to_f32(uint32_t bits16) {
  if constexpr (DT == HR_BF16) {
    return __uint_as_float(bits16 << 16);
  } else {
    return __half2float(__ushort_as_half((unsigned short)bits16));
  }
}
// 8 16-bit source elements -> fp32 pairs (element 2i in .x)
template <int DT>
__device__ __forceinline__ void unpack8(const uint4& raw, float2 (&x)[4]) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (DT == HR_BF16) {
      x[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
    } else {
      x[i] = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    }
  }
}
// magnitude bit patterns, max over the 8 values (NaN/Inf on top); 16-bit patterns in both halves
__device__ __forceinline__ uint32_t absmax_pair(const uint4& raw) {
  const uint32_t m = 0x7FFF7FFFu;
  return __vmaxu2(__vmaxu2(raw.x & m, raw.y & m), __vmaxu2(raw.z & m, raw.w & m));
}
template <int DT>
__device__ __forceinline__ bool pattern_nonfinite(uint32_t pair_max) {
  const uint32_t v = max(pair_max & 0xFFFFu, pair_max >> 16);
  return v >= (DT == HR_BF16 ? 0x7F80u : 0x7C00u);
}
// bytes 0 of four words -> one word
__device__ __forceinline__ uint32_t gather_b0(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// bytes 3 of four words -> one word
__device__ __forceinline__ uint32_t gather_b3(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0073), __byte_perm(c, d, 0x0073), 0x5410);
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

// fl(d / 15) for the INT4 scale, the same correction with y = RN(1/15): checked against __fdiv_rn for every
// fp32 significand at every exponent from 2^-100 to 2^127 by tests/csrc/markstein_check.cu (the quotient
// of a power-of-two scaled d is the scaled quotient while the residual cannot underflow); smaller d take
// the IEEE division.
__device__ __forceinline__ float div15(float d) {
  constexpr float y = 0.066666670143604278564f;  // RN(1/15)
  if (d < 7.8886090522101181e-31f) return __fdiv_rn(d, 15.f);
  const float q0 = __fmul_rn(d, y);
  const float r = __fmaf_rn(-q0, 15.f, d);
  return __fmaf_rn(r, y, q0);
}

// sub(a, b) of R4: fl(a - b) saturated at FLT_MAX (finite inputs whose difference overflows)
__device__ __forceinline__ float sub_sat(float a, float b) { return fminf(__fsub_rn(a, b), 3.40282347e+38f); }

// ------------------------------------------------------------------ INT8 / INT4 (G <= 256)
// A warp step covers 1024 consecutive elements; lane L owns the 32 elements [32L, 32L + 32), so a
// group of G is SEGL = G/32 lanes: the per-lane statistics are plain min/max chains, the cross-lane
// reduction is log2(SEGL) <= 3 shuffles, and the group scalars are computed by SEGL lanes only.
// Shared-memory reads: the lane's four 16-B chunks are read in the rotated order
// c = (j + (L >> 1)) & 3, which makes every quarter-warp load cover 32 distinct banks; the codes are
// rotated back in registers before the 16-B stores.
constexpr uint32_t kStep = 1024;  // elements per warp step
constexpr uint32_t kLaneE = 32;   // elements per lane and step

template <int DT>
__device__ __forceinline__ bool load_lane32(const uint8_t* tile, uint32_t e0, uint32_t n_el, uint32_t rot,
                                            uint4 (&raw)[4]) {
  const bool valid = e0 < n_el;  // n_el is a multiple of 256: a lane's 32 elements are all valid or none
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j)
    raw[j] = valid ? *reinterpret_cast<const uint4*>(tile + 2 * (e0 + ((j + rot) & 3) * 8)) : make_uint4(0, 0, 0, 0);
  return valid;
}
// slot j holds chunk (j + rot) & 3: put chunk c back at position c
template <class V>
__device__ __forceinline__ void unrotate4(V (&w)[4], uint32_t rot) {
  if (rot & 1) {
    const V t = w[3];
    w[3] = w[2], w[2] = w[1], w[1] = w[0], w[0] = t;
  }
  if (rot & 2) {
    V t = w[0];
    w[0] = w[2], w[2] = t;
    t = w[1];
    w[1] = w[3], w[3] = t;
  }
}

// a3: a = max |x| (exact: the largest magnitude bit pattern); s = 1 if a == 0 else fl(a / 127).
// a4: q = rne(fl(x / s)) with fl(x/s) by Markstein's correction, y = RN(1/s): equal to the IEEE quotient
// for every (a, x) pair of 16-bit values when s is in [2^-90, 2^125] (tests/csrc/markstein_check.cu,
// exhaustive); outside that range the IEEE division.  |x| <= a gives |x/s| <= 127 (1 + 2^-24), so the
// clamp to [-127, 127] never binds and is omitted; rne comes from fl(v + 1.5*2^23), whose low byte is
// the two's-complement code.
template <int SEGL, int DT>
__device__ __forceinline__ void enc_int8_step(const uint8_t* tile, uint32_t eb, uint32_t n_el, uint8_t* codes,
                                              float* meta, uint32_t g_shift, uint32_t lane, uint32_t& nan_acc) {
  const uint32_t e0 = eb + lane * kLaneE, rot = (lane >> 1) & 3;
  uint4 raw[4];
  const bool valid = load_lane32<DT>(tile, e0, n_el, rot, raw);
  const uint32_t pm = __vmaxu2(__vmaxu2(absmax_pair(raw[0]), absmax_pair(raw[1])),
                               __vmaxu2(absmax_pair(raw[2]), absmax_pair(raw[3])));
  const uint32_t ab = seg_max_u32<SEGL>(max(pm & 0xFFFFu, pm >> 16));
  nan_acc = __vmaxu2(nan_acc, ab);  // NaN/Inf
  const float a = to_f32<DT>(ab);
  const float s = (a == 0.f) ? 1.f : div127(a);
  if ((lane & (SEGL - 1)) == 0 && valid) meta[e0 >> g_shift] = s;
  const bool fast = s >= 8.0779356e-28f && s <= 4.2535296e+37f;
  uint2 w[4];
  if (__all_sync(0xFFFFFFFFu, fast)) {  // warp-uniform: the branch-free path for every normal scale
    const float y = __frcp_rn(s);  // RN(1/s)
    const float2 yy = make_float2(y, y), ns = make_float2(-s, -s), mg = make_float2(kMagic, kMagic);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 x[4];
      unpack8<DT>(raw[j], x);
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 q0 = __fmul2_rn(x[i], yy);
        const float2 qf = __ffma2_rn(__ffma2_rn(q0, ns, x[i]), yy, q0);  // fl(x / s)
        const float2 rr = __fadd2_rn(qf, mg);
        v[2 * i] = __float_as_uint(rr.x), v[2 * i + 1] = __float_as_uint(rr.y);
      }
      w[j] = make_uint2(gather_b0(v[0], v[1], v[2], v[3]), gather_b0(v[4], v[5], v[6], v[7]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 x[4];
      unpack8<DT>(raw[j], x);
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[2 * i] = (uint32_t)__float2int_rn(__fdiv_rn(x[i].x, s));
        v[2 * i + 1] = (uint32_t)__float2int_rn(__fdiv_rn(x[i].y, s));
      }
      w[j] = make_uint2(gather_b0(v[0], v[1], v[2], v[3]), gather_b0(v[4], v[5], v[6], v[7]));
    }
  }
  unrotate4(w, rot);
  if (valid) {
    uint4* dst = reinterpret_cast<uint4*>(codes + e0);
    dst[0] = make_uint4(w[0].x, w[0].y, w[1].x, w[1].y);
    dst[1] = make_uint4(w[2].x, w[2].y, w[3].x, w[3].y);
  }
}

// a3: mn = min + 0, mx = max + 0 (a zero extreme is +0); s = (mx == mn) ? 1 : fl(sub(mx, mn) / 15).
// a4: q = clamp(rne(fl(sub(x, mn) / s)), 0, 15); element 2i -> low nibble (R24).  u = sub(x, mn) is in
// [0, sub(mx, mn)], so fl(u / s) is in [0, 15 (1 + 2^-23)] and the clamp never binds.  fl(u / s) without
// a division: y = RN(1/s), q0 = RN(u*y) (within 2 ulps), one Markstein correction q1 = RN(q0 + r0*y),
// r0 = u - s*q0 (FMA), makes q1 faithful, and a second one, q2 = RN(q1 + r1*y), is the correctly
// rounded quotient (Markstein's theorem: y within 1/2 ulp of 1/s, q1 within 1 ulp of u/s).  Checked
// against IEEE division on 2^33 sampled (x, mn, mx) triples per source dtype by
// tests/csrc/markstein_check.cu.  Scales outside [2^-90, 2^125] (or a group whose range overflows) take
// __fdiv_rn per element (warp-uniform).
// Packed 16-bit min / NaN-propagating max of two source-dtype pairs (HMNMX2): the order of bf16 / fp16
// values is the order of their fp32 images, so the extremes equal the fp32 ones up to the sign of a zero
// (made +0 by the caller's fl(v + 0)).
template <int DT>
__device__ __forceinline__ uint32_t pmin16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  if constexpr (DT == HR_BF16) asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  else asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <int DT>
__device__ __forceinline__ uint32_t pmaxnan16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  if constexpr (DT == HR_BF16) asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  else asm("max.NaN.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <int SEGL, int DT>
__device__ __forceinline__ void enc_int4_step(const uint8_t* tile, uint32_t eb, uint32_t n_el, uint8_t* codes,
                                              float2* meta, uint32_t g_shift, uint32_t lane, uint32_t& nan_acc) {
  const uint32_t e0 = eb + lane * kLaneE, rot = (lane >> 1) & 3;
  uint4 raw[4];
  const bool valid = load_lane32<DT>(tile, e0, n_el, rot, raw);
  // lane statistics on the packed pairs: min, and a NaN-propagating max, so that the lane's NaN / +-Inf
  // show up as a non-finite pattern in one of the two (a NaN in max, +Inf in max, -Inf in min)
  // (a pairwise tree: 4 dependent levels instead of a 15-long chain)
  uint32_t tmn[8], tmx[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    tmn[2 * j] = pmin16x2<DT>(raw[j].x, raw[j].y), tmx[2 * j] = pmaxnan16x2<DT>(raw[j].x, raw[j].y);
    tmn[2 * j + 1] = pmin16x2<DT>(raw[j].z, raw[j].w), tmx[2 * j + 1] = pmaxnan16x2<DT>(raw[j].z, raw[j].w);
  }
#pragma unroll
  for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) tmn[i] = pmin16x2<DT>(tmn[i], tmn[i + w]), tmx[i] = pmaxnan16x2<DT>(tmx[i], tmx[i + w]);
  const uint32_t pmn = tmn[0], pmx = tmx[0];
  nan_acc = __vmaxu2(nan_acc, __vmaxu2(pmn & 0x7FFF7FFFu, pmx & 0x7FFF7FFFu));
  float2 x[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack8<DT>(raw[j], x[j]);
  float mn = fminf(to_f32<DT>(pmn & 0xFFFFu), to_f32<DT>(pmn >> 16));
  float mx = fmaxf(to_f32<DT>(pmx & 0xFFFFu), to_f32<DT>(pmx >> 16));
  mn = __fadd_rn(seg_min_f<SEGL>(mn), 0.f);
  mx = __fadd_rn(seg_max_f<SEGL>(mx), 0.f);
  const float dm = __fsub_rn(mx, mn);
  const float s = (mx == mn) ? 1.f : div15(fminf(dm, 3.40282347e+38f));
  if ((lane & (SEGL - 1)) == 0 && valid) meta[e0 >> g_shift] = make_float2(s, mn);
  const bool fast = s >= 8.0779356e-28f && s <= 4.2535296e+37f && dm <= 3.40282347e+38f;
  uint32_t w[4];
  if (__all_sync(0xFFFFFFFFu, fast)) {  // warp-uniform
    const float y = __frcp_rn(s);  // RN(1/s)
    const float2 yy = make_float2(y, y), ns = make_float2(-s, -s), nm = make_float2(-mn, -mn);
    const float2 mg = make_float2(kMagic, kMagic);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 u = __fadd2_rn(x[j][i], nm);
        const float2 q0 = __fmul2_rn(u, yy);
        const float2 q1 = __ffma2_rn(__ffma2_rn(q0, ns, u), yy, q0);
        const float2 q2 = __ffma2_rn(__ffma2_rn(q1, ns, u), yy, q1);  // fl(u / s)
        const float2 rr = __fadd2_rn(q2, mg);                          // low bits: rne, in [0, 15]
        // even element -> low nibble, odd -> high nibble: the low byte of lo + (hi << 4) (one LEA)
        v[i] = __float_as_uint(rr.x) + (__float_as_uint(rr.y) << 4);
      }
      w[j] = gather_b0(v[0], v[1], v[2], v[3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = (uint32_t)__float2int_rn(__fdiv_rn(sub_sat(i & 1 ? x[j][i >> 1].y : x[j][i >> 1].x, mn), s));
      w[j] = (gather_b0(v[0], v[2], v[4], v[6]) & 0x0F0F0F0Fu) | ((gather_b0(v[1], v[3], v[5], v[7]) & 0x0F0F0F0Fu) << 4);
    }
  }
  unrotate4(w, rot);
  if (valid) *reinterpret_cast<uint4*>(codes + e0 / 2) = make_uint4(w[0], w[1], w[2], w[3]);
}

// ------------------------------------------------------------------ FP8 (nearest, ties to even, saturating: R5)
template <int SCHEME, int DT>
__device__ __forceinline__ void enc_fp8(const uint4& raw, uint8_t* codes, uint32_t e, uint32_t& nan_acc) {
  constexpr __nv_fp8_interpretation_t kInterp = SCHEME == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
  nan_acc = __vmaxu2(nan_acc, absmax_pair(raw));
  float2 x[4];
  unpack8<DT>(raw, x);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = __nv_cvt_float2_to_fp8x2(x[i], __NV_SATFINITE, kInterp);
  *reinterpret_cast<uint2*>(codes + e) = make_uint2(__byte_perm(c[0], c[1], 0x5410), __byte_perm(c[2], c[3], 0x5410));
}

// ------------------------------------------------------------------ MXFP8 (R31)
// A 32-element block = the 8 elements of each of 4 consecutive lanes.  Block max |x| from 16-bit magnitude
// patterns (two shuffles), e = max(ef(max) - 127 - 8, -127) (ef = 0, a zero block or an fp32-subnormal
// maximum: -127), elements = satfinite RNE E4M3 of x * 2^-e (exact: |x * 2^-e| < 512, and below 2^-126 the
// E4M3 rounding is 0 either way), scale byte e + 127 written by the block's first lane.
template <int DT>
__device__ __forceinline__ void enc_mxfp8(const uint4& raw, uint8_t* codes, uint8_t* scales, uint32_t e,
                                          uint32_t lane, uint32_t& nan_acc) {
  const uint32_t pm = absmax_pair(raw);
  nan_acc = __vmaxu2(nan_acc, pm);
  uint32_t am = max(pm & 0xFFFFu, pm >> 16);
  am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, 1));
  am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, 2));
  const uint32_t ef = DT == HR_BF16 ? (am >> 7) : ((__float_as_uint(__half2float(__ushort_as_half((unsigned short)am))) >> 23) & 0xFFu);
  const int ex = ef == 0 ? -127 : max((int)ef - 135, -127);
  const float inv = __uint_as_float((uint32_t)(127 - ex) << 23);  // 2^-e, a normal fp32 (127 - e in [8, 254])
  float2 x[4];
  unpack8<DT>(raw, x);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    c[i] = __nv_cvt_float2_to_fp8x2(__fmul2_rn(x[i], make_float2(inv, inv)), __NV_SATFINITE, __NV_E4M3);
  *reinterpret_cast<uint2*>(codes + e) = make_uint2(__byte_perm(c[0], c[1], 0x5410), __byte_perm(c[2], c[3], 0x5410));
  if ((lane & 3) == 0) scales[e >> 5] = (uint8_t)(ex + 127);
}

// ------------------------------------------------------------------ GSE-8
// Table entry per fp32 biased exponent ef of the slab (built by the producer warp):
//   bits 24..30 and 8..14   idx << m   (idx: smallest G_i >= E)
//   bits 31 and 15          1 (sign kept) — 0 for codes that flush (zero, subnormal, E below the array's reach)
//   bits 0..4               31 - keep  keep = m - 1 - d fraction bits after the marker, d = G_idx - E
// The code of x (fp32 bits b) is byte 3 of ((b | 0x7FFFFFFF) & ent) | ({m24 : 0} >> (31 - keep)), with
// m24 = 1.fraction (24 bits): the funnel shift puts the marker 1 and the top keep fraction bits (the
// rest truncated, R9) in byte 3 below idx.  A flushed entry is 0: both terms vanish.  For a bf16 pair
// word w the high element is exactly that with b = w; the low element assembles its code in byte 1
// ((w | 0xFFFF7FFF) & ent keeps its sign bit 15, and {m8 : 0} >> (31 - keep) with m8 = 1.fraction
// (8 bits) puts the field in byte 1), so no unpacking to fp32 is needed.
template <int DT>
__device__ __forceinline__ void enc_gse(const uint4& raw, uint8_t* codes, uint32_t tab, uint32_t e,
                                        uint32_t& nan_acc) {
  nan_acc = __vmaxu2(nan_acc, absmax_pair(raw));
  uint32_t c[8];
  if constexpr (DT == HR_BF16) {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t eh = lds32(tab | ((w[i] >> 21) & 0x3FCu));
      const uint32_t el = lds32(tab | ((w[i] >> 5) & 0x3FCu));
      c[2 * i + 1] = ((w[i] | 0x7FFFFFFFu) & eh) | __funnelshift_r(0u, (w[i] & 0x007F0000u) | 0x00800000u, eh);
      c[2 * i] = ((w[i] | 0xFFFF7FFFu) & el) | __funnelshift_r(0u, (w[i] & 0x7Fu) | 0x80u, el);
    }
    *reinterpret_cast<uint2*>(codes + e) = make_uint2(__byte_perm(__byte_perm(c[0], c[1], 0x0071), __byte_perm(c[2], c[3], 0x0071), 0x5410),
                                                      __byte_perm(__byte_perm(c[4], c[5], 0x0071), __byte_perm(c[6], c[7], 0x0071), 0x5410));
  } else {
    float2 x[4];
    unpack8<DT>(raw, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t b = __float_as_uint(i & 1 ? x[i >> 1].y : x[i >> 1].x);
      const uint32_t ent = lds32(tab | ((b >> 21) & 0x3FCu));
      c[i] = ((b | 0x7FFFFFFFu) & ent) | __funnelshift_r(0u, (b & 0x007FFFFFu) | 0x00800000u, ent);
    }
    *reinterpret_cast<uint2*>(codes + e) = make_uint2(gather_b3(c[0], c[1], c[2], c[3]), gather_b3(c[4], c[5], c[6], c[7]));
  }
}

// the slab's array parameters from its exponent range (rule C, R6): lo, Emax, n entries
struct GseArr {
  int lo, Emax, n, rmin, rmax;  // rmin / rmax: biased exponent range of the slab's nonzero normals
};
__device__ __forceinline__ GseArr gse_array(const int* range, int m, int nmax) {
  const int step = m - 1;
  const int rmin = 255 - range[0], rmax = range[1];
  GseArr a;
  a.Emax = rmax - 127;
  a.lo = max(rmin - 127, a.Emax - (nmax - 1) * step);
  a.n = rmax != 0 ? (a.Emax - a.lo + step - 1) / step + 1 : 0;
  a.rmin = rmin, a.rmax = rmax;
  return a;
}

// producer warp: the code-template table of one slab.  Only exponents that occur in the slab
// ([rmin, rmax], and 0 for zeros / subnormals) are written; other entries are never read (a NaN/Inf
// input, ef = 255, is rejected through the error flag).
__device__ __forceinline__ void gse_build_table(uint32_t* tab, const GseArr& a, int m, int lane) {
  const int step = m - 1;
  if (lane == 0) tab[0] = 0u;
  if (a.n == 0) return;
  for (int ef = a.rmin + lane; ef <= min(a.rmax, 254); ef += 32) {
    const int E = ef - 127;
    const int idx = (E <= a.lo) ? 0 : (E - a.lo + step - 1) / step;
    const int d = min(a.lo + idx * step, a.Emax) - E;
    uint32_t ent = 0;
    if (d <= m - 1) {
      const uint32_t t = 0x80u | ((uint32_t)idx << m);  // sign enable | idx << m
      ent = (t << 24) | (t << 8) | (uint32_t)(31 - (m - 1 - d));
    }
    tab[ef] = ent;
  }
}

// producer warp: the slab's meta record — int8 array [2^e] (unused -128), zero pad to 16 B, then the fp32
// decode table [2^(e+1)]: entry (sign << e | i) = (-1)^sign 2^(G_i - (m-1)), 0 for unused i
__device__ __forceinline__ void gse_write_record(uint8_t* meta, uint32_t stride, const GseArr& a, int m, int nmax,
                                                 int lane) {
  const int step = m - 1;
  if (lane < 16) {
    int v = 0;
    if (lane < nmax) v = (lane < a.n) ? min(a.lo + lane * step, a.Emax) : -128;
    meta[lane] = (uint8_t)(int8_t)v;
  }
  for (uint32_t w = lane; w < (stride - 16) / 4; w += 32) {
    float v = 0.f;
    const int i = (int)w & (nmax - 1);
    if ((int)w < 2 * nmax && i < a.n) {
      const int k = min(a.lo + i * step, a.Emax) - step;
      v = k >= -126 ? __int_as_float((k + 127) << 23) : (k >= -149 ? __int_as_float(1 << (k + 149)) : 0.f);
      if ((int)w >= nmax) v = -v;
    }
    reinterpret_cast<float*>(meta + 16)[w] = v;
  }
}

// ------------------------------------------------------------------ producer
template <int MODE>
__device__ __forceinline__ void q_produce(const QBatch& p, const QSmem& sm, int lane) {
  const uint32_t per_job = p.L * p.Hl * p.tiles_per_slab;
  const int m = (int)p.gse_m, nmax = 1 << (7 - m);
  uint64_t i = 0;  // stage sequence number across this CTA's ranges
  auto range = [&](uint64_t t0, uint64_t t1) {
    if (t1 <= t0) return;
    uint32_t j = (uint32_t)(t0 / per_job);
    uint32_t r = (uint32_t)(t0 - (uint64_t)j * per_job);
    uint32_t slab_i = r / p.tiles_per_slab, sub = r - slab_i * p.tiles_per_slab;
    uint32_t l = slab_i / p.Hl, hl = slab_i - l * p.Hl;
    for (uint64_t t = t0; t < t1; ++t, ++i) {
      const int stage = (int)(i % kQStages);
      if (i >= kQStages) mbar_wait(&sm.empty()[stage], (uint32_t)(((i / kQStages) - 1) & 1));
      const QJob& jb = p.jobs[j];
      const uint32_t scheme = jb.scheme;
      const uint32_t e0 = sub * p.tile_e;
      const uint32_t n_el = min(p.tile_e, p.slab - e0);
      uint8_t* meta = jb.dst + p.meta_off[scheme] + (uint64_t)slab_i * p.meta_stride[scheme];
      if (MODE == MODE_ENCODE && scheme == HR_S_GSE8) {
        const GseArr a = gse_array(jb.range + 2 * slab_i, m, nmax);
        gse_build_table(sm.gtab(stage), a, m, lane);
        if (sub == 0) gse_write_record(meta, p.meta_stride[HR_S_GSE8], a, m, nmax, lane);
        __syncwarp();
      }
      if (lane == 0) {
        QHdr& h = sm.hdr()[stage];
        h.codes = jb.dst + (uint64_t)slab_i * p.code_slab[scheme] + code_bytes(scheme, e0);
        h.meta = scheme == HR_S_INT8 ? meta + 4 * (e0 >> p.g_shift) : scheme == HR_S_INT4 ? meta + 8 * (e0 >> p.g_shift)
             : scheme == HR_S_MXFP8 ? meta + (e0 >> 5) : meta;
        h.range = jb.range ? jb.range + 2 * slab_i : nullptr;
        h.n_el = n_el;
        h.scheme = scheme;
        uint64_t* full = &sm.full()[stage];
        mbar_arrive_expect_tx(full, 2 * n_el);  // release: header and table visible with the phase flip
        bulk_g2s(sm.tile(stage), jb.src + ((uint64_t)(l * p.H + p.h0 + hl) * p.slab + e0), 2 * n_el, full);
      }
      if (++sub == p.tiles_per_slab) {  // advance (sub, head, layer, job) without divisions
        sub = 0;
        ++slab_i;
        if (++hl == p.Hl) {
          hl = 0;
          if (++l == p.L) l = 0, slab_i = 0, ++j;
        }
      }
    }
  };
  const uint64_t ns = p.sched ? p.n_tiles - p.dyn_tiles : p.n_tiles;
  range(ns * blockIdx.x / gridDim.x, ns * (blockIdx.x + 1) / gridDim.x);
  if (p.sched) {
    while (true) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(reinterpret_cast<unsigned long long*>(p.sched), (unsigned long long)p.dyn_chunk);
      c = __shfl_sync(0xFFFFFFFFu, c, 0);
      if (c >= p.dyn_tiles) break;
      const uint64_t ce = c + p.dyn_chunk < p.dyn_tiles ? c + p.dyn_chunk : p.dyn_tiles;
      range(ns + c, ns + ce);
    }
    const int stage = (int)(i % kQStages);  // end marker: a header with n_el = 0
    if (i >= kQStages) mbar_wait(&sm.empty()[stage], (uint32_t)(((i / kQStages) - 1) & 1));
    if (lane == 0) {
      sm.hdr()[stage].n_el = 0;
      mbar_arrive(&sm.full()[stage]);
      __threadfence();
      if (atomicAdd(reinterpret_cast<unsigned int*>(p.sched) + 2, 1u) == gridDim.x - 1) {
        *reinterpret_cast<volatile unsigned long long*>(p.sched) = 0ull;
        reinterpret_cast<volatile unsigned int*>(p.sched)[2] = 0u;
      }
    }
  }
}

// ------------------------------------------------------------------ consumers
// Encode one staged tile: warp cw of NW consumer warps takes every NW-th 256-element chunk / 1024-element
// step.  PASS16 is written back by the bulk-copy engine (issued by warp 0 lane 0, waited before return).
template <int DT, int SEG, int NW>
__device__ __forceinline__ void encode_tile(const QBatch& p, const QHdr& h, const uint8_t* tile, uint32_t gtab_addr,
                                            int cw, int lane, uint32_t& nan_acc) {
  const uint32_t n_ch = h.n_el / kChunk;
  switch (h.scheme) {
    case HR_S_PASS16:
      if (cw == 0 && lane == 0) bulk_s2g(h.codes, tile, 2 * h.n_el);
      for (uint32_t c = cw; c < n_ch; c += NW)
        nan_acc = __vmaxu2(nan_acc, absmax_pair(*reinterpret_cast<const uint4*>(tile + 2 * (c * kChunk + lane * 8))));
      if (cw == 0 && lane == 0) bulk_wait_read_all();  // the stage may be reused after this
      break;
    case HR_S_INT8:
      for (uint32_t eb = cw * kStep; eb < h.n_el; eb += NW * kStep)
        enc_int8_step<SEG / 4, DT>(tile, eb, h.n_el, h.codes, reinterpret_cast<float*>(h.meta), p.g_shift, lane,
                                   nan_acc);
      break;
    case HR_S_INT4:
      for (uint32_t eb = cw * kStep; eb < h.n_el; eb += NW * kStep)
        enc_int4_step<SEG / 4, DT>(tile, eb, h.n_el, h.codes, reinterpret_cast<float2*>(h.meta), p.g_shift, lane,
                                   nan_acc);
      break;
    case HR_S_FP8E4M3:
#pragma unroll 2
      for (uint32_t c = cw; c < n_ch; c += NW) {
        const uint32_t e = c * kChunk + lane * 8;
        enc_fp8<HR_S_FP8E4M3, DT>(*reinterpret_cast<const uint4*>(tile + 2 * e), h.codes, e, nan_acc);
      }
      break;
    case HR_S_FP8E5M2:
#pragma unroll 2
      for (uint32_t c = cw; c < n_ch; c += NW) {
        const uint32_t e = c * kChunk + lane * 8;
        enc_fp8<HR_S_FP8E5M2, DT>(*reinterpret_cast<const uint4*>(tile + 2 * e), h.codes, e, nan_acc);
      }
      break;
    case HR_S_GSE8:
#pragma unroll 2
      for (uint32_t c = cw; c < n_ch; c += NW) {
        const uint32_t e = c * kChunk + lane * 8;
        enc_gse<DT>(*reinterpret_cast<const uint4*>(tile + 2 * e), h.codes, gtab_addr, e, nan_acc);
      }
      break;
    case HR_S_MXFP8:  // h.meta: the tile's first scale byte
#pragma unroll 2
      for (uint32_t c = cw; c < n_ch; c += NW) {
        const uint32_t e = c * kChunk + lane * 8;
        enc_mxfp8<DT>(*reinterpret_cast<const uint4*>(tile + 2 * e), h.codes, h.meta, e, lane, nan_acc);
      }
      break;
    default:
      break;
  }
}

template <int DT, int SEG>
__device__ __forceinline__ void q_consume_encode(const QBatch& p, const QSmem& sm, int cw, int lane) {
  const uint64_t ns = p.sched ? p.n_tiles - p.dyn_tiles : p.n_tiles;
  const uint64_t t0 = ns * blockIdx.x / gridDim.x, t1 = ns * (blockIdx.x + 1) / gridDim.x;
  uint32_t nan_acc = 0;
  for (uint64_t i = 0; p.sched || i < t1 - t0; ++i) {
    const int stage = (int)(i % kQStages);
    mbar_wait(&sm.full()[stage], (uint32_t)((i / kQStages) & 1));
    const QHdr h = sm.hdr()[stage];
    if (h.n_el == 0) break;  // the producer's end marker (tail-balanced launches)
    // GSE-8 table: 1-KB aligned, entry address = tab | 4*ef
    encode_tile<DT, SEG, kQWarps>(p, h, sm.tile(stage), smem_addr(sm.gtab(stage)), cw, lane, nan_acc);
    __syncwarp();
    if (lane == 0) mbar_arrive_relaxed(&sm.empty()[stage]);
  }
  if (cw == 0 && lane == 0) bulk_wait_all();
  if (pattern_nonfinite<DT>(nan_acc)) atomicOr(p.err, 1);
}

// Non-persistent variant for schemes without a slab-wide dependency (INT8, INT4, FP8, PASS16): one CTA of
// kTileWarps warps per tile, one TMA copy of the tile's source, encode, exit — many small CTAs per SM
// overlap their copies with each other's encode.
constexpr int kTileWarps = 8;
template <int DT, int SEG>
__global__ void __launch_bounds__(32 * kTileWarps) quant_tile_kernel(const __grid_constant__ QBatch p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  uint8_t* tile = smem_raw + 128;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t per_job = p.L * p.Hl * p.tiles_per_slab;
  const uint32_t t = blockIdx.x, j = t / per_job, r = t - j * per_job;
  const uint32_t slab_i = r / p.tiles_per_slab, sub = r - slab_i * p.tiles_per_slab;
  const uint32_t l = slab_i / p.Hl, hl = slab_i - l * p.Hl;
  const QJob& jb = p.jobs[j];
  const uint32_t scheme = jb.scheme, e0 = sub * p.tile_e, n_el = min(p.tile_e, p.slab - e0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init_fence();
    mbar_arrive_expect_tx(bar, 2 * n_el);
    bulk_g2s(tile, jb.src + ((uint64_t)(l * p.H + p.h0 + hl) * p.slab + e0), 2 * n_el, bar);
  }
  QHdr h;
  uint8_t* meta = jb.dst + p.meta_off[scheme] + (uint64_t)slab_i * p.meta_stride[scheme];
  h.codes = jb.dst + (uint64_t)slab_i * p.code_slab[scheme] + code_bytes(scheme, e0);
  h.meta = scheme == HR_S_INT8 ? meta + 4 * (e0 >> p.g_shift) : scheme == HR_S_INT4 ? meta + 8 * (e0 >> p.g_shift)
             : scheme == HR_S_MXFP8 ? meta + (e0 >> 5) : meta;
  h.range = nullptr;
  h.n_el = n_el;
  h.scheme = scheme;
  __syncthreads();  // barrier initialised before anyone waits on it
  mbar_wait(bar, 0);
  uint32_t nan_acc = 0;
  encode_tile<DT, SEG, kTileWarps>(p, h, tile, 0u, warp, lane, nan_acc);
  if (warp == 0 && lane == 0) bulk_wait_all();
  if (pattern_nonfinite<DT>(nan_acc)) atomicOr(p.err, 1);
}

// RANGE mode: per-slab min / max biased fp32 exponent over nonzero normal values (R8, R9).
// bf16: from 16-bit patterns two at a time — max magnitude pattern -> Emax; for Emin the key
// (mag + 0x7F80) ^ 0x8000 maps normals (mag >= 0x80) to mag - 0x80 and zeros / subnormals above 0x7FFF,
// so the minimum key is the smallest normal.  fp16: per element in fp32 (fp16 subnormals are fp32
// normals).
template <int DT>
__device__ __forceinline__ void q_consume_range(const QBatch& p, const QSmem& sm, int cw, int lane) {
  const uint64_t ns = p.sched ? p.n_tiles - p.dyn_tiles : p.n_tiles;
  const uint64_t t0 = ns * blockIdx.x / gridDim.x, t1 = ns * (blockIdx.x + 1) / gridDim.x;
  bool bad = false;
  int emin = 255, emax = 0;  // running range of the current slab (this warp's chunks)
  int* cur = nullptr;
  auto flush = [&] {  // warp-reduce and publish the running range of slab `cur`
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
    }
    if (lane == 0 && emax != 0) {  // stored as (255 - min, max) so a zero fill initialises it
      atomicMax(&cur[0], 255 - emin);
      atomicMax(&cur[1], emax);
    }
    emin = 255, emax = 0;
  };
  for (uint64_t i = 0; p.sched || i < t1 - t0; ++i) {
    const int stage = (int)(i % kQStages);
    mbar_wait(&sm.full()[stage], (uint32_t)((i / kQStages) & 1));
    const QHdr h = sm.hdr()[stage];
    if (h.n_el == 0) break;
    const uint8_t* tile = sm.tile(stage);
    const uint32_t n_ch = h.n_el / kChunk;
    if (h.range != cur) {
      if (cur) flush();
      cur = h.range;
    }
    if constexpr (DT == HR_BF16) {
      uint32_t mx = 0u, mn = 0xFFFFFFFFu;
      for (uint32_t c = cw; c < n_ch; c += kQWarps) {
        const uint4 raw = *reinterpret_cast<const uint4*>(tile + 2 * (c * kChunk + lane * 8));
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t mag = w[k] & 0x7FFF7FFFu;
          mx = __vmaxu2(mx, mag);
          mn = __vminu2(mn, (mag + 0x7F807F80u) ^ 0x80008000u);
        }
      }
      const uint32_t pmax = max(mx & 0xFFFFu, mx >> 16), kmin = min(mn & 0xFFFFu, mn >> 16);
      bad |= pmax >= 0x7F80u;
      emax = max(emax, (int)(pmax >> 7));
      if (kmin < 0x8000u) emin = min(emin, (int)((kmin + 0x80u) >> 7));
    } else {
      for (uint32_t c = cw; c < n_ch; c += kQWarps) {
        const uint4 raw = *reinterpret_cast<const uint4*>(tile + 2 * (c * kChunk + lane * 8));
        float2 x[4];
        unpack8<DT>(raw, x);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t b = __float_as_uint(k & 1 ? x[k >> 1].y : x[k >> 1].x);
          const int ef = (b >> 23) & 0xFF;
          bad |= ef == 255;
          if (ef != 0) emin = min(emin, ef), emax = max(emax, ef);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_relaxed(&sm.empty()[stage]);
  }
  if (cur) flush();
  if (bad) atomicOr(p.err, 1);
}

template <int DT, int SEG, int MODE>
__global__ void __launch_bounds__(kQThreadsB, 1) quantize_batch_kernel(const __grid_constant__ QBatch p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const QSmem sm{smem_raw};
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    if (smem_addr(smem_raw) & 1023u) __trap();  // GSE-8 table addressing (tab | 4*ef) needs 1-KB alignment
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&sm.full()[s], 1);
      mbar_init(&sm.empty()[s], kQWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();
  if (warp == 0) {
    q_produce<MODE>(p, sm, lane);
  } else if (MODE == MODE_RANGE) {
    q_consume_range<DT>(p, sm, warp - 1, lane);
  } else {
    q_consume_encode<DT, SEG>(p, sm, warp - 1, lane);
  }
}

// ---------------------------------------------------------------- GSE-8, single pass: a slab per cluster
// A cluster of kGseQ CTAs owns one (item, layer, head) slab (default 2: halves); CTA q bulk-copies part q of the slab's
// source into its shared memory (one TMA copy), computes the quarter's exponent range, writes it into
// every peer's shared memory (DSMEM, st.shared::cluster), and after one cluster barrier each CTA has
// the slab-wide range, builds the code-template table (one entry per thread) and encodes its quarter
// from shared memory.  The source is read from HBM once; many small CTAs per SM overlap the copies
// with the encode.  Used when a quarter slab fits kGseQMaxBytes (every Llama shape).
// cluster size / threads / resident CTAs measured (tools/prof_quant.py GSE8 64, profiles/round2/tuning.md):
// 2 x 256 threads 11.05-11.40 us/item; 4 x 128 (round 1) 12.38-12.52; 2 x 128 11.71-12.06; 2 x 512 11.73-11.81;
// 4 x 256 12.24-12.33; 8 x 128 12.85-12.88; 1 x 256 / 512 (no cluster, one CTA per SM) 14.2-14.4
#ifndef HARAG_GSE_Q
#define HARAG_GSE_Q 2
#endif
#ifndef HARAG_GSE_MINB
#define HARAG_GSE_MINB 3
#endif
constexpr int kGseQ = HARAG_GSE_Q;        // CTAs per cluster (= slab parts; "quarters" at the default 4)
#ifndef HARAG_GSE_THREADS
#define HARAG_GSE_THREADS 256
#endif
constexpr int kGseThreads = HARAG_GSE_THREADS;  // 128 elements per thread at Llama shapes: amortises the per-slab setup
#ifndef HARAG_GSE_QMAX_KB
#define HARAG_GSE_QMAX_KB 64
#endif
constexpr uint32_t kGseQMaxBytes = HARAG_GSE_QMAX_KB * 1024;
constexpr uint32_t kGseHdr = 8192;  // table + exchange + barrier

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// {a, b} into CTA `rank`'s shared memory at the image of local_addr; the store completes 8 bytes of the
// transaction count of that CTA's mbarrier at the image of local_bar (DSMEM st.async: the receiver waits on
// its own mbarrier instead of a release/acquire cluster barrier)
__device__ __forceinline__ void st_async_cluster_v2(uint32_t local_addr, uint32_t local_bar, uint32_t rank, int a, int b) {
  uint32_t remote, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(local_bar), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s32 [%0], {%1, %2}, [%3];"
               ::"r"(remote), "r"(a), "r"(b), "r"(rbar) : "memory");
}

// (a & imm) | b with b a register (one LOP3; the compiler would spend two with two immediates)
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(0x007F007Fu), "r"(b));  // (a & b) | c
  return d;
}
// GSE-8 codes of 8 bf16 values with a 512-entry table indexed by sign|exponent (9 bits): the entry of a
// negative value already carries its sign bit (bits 31 and 15), so the code of the high bf16 of a word w
// is byte 3 of ent | ({1.fraction : 0} >> (31 - keep)), of the low bf16 byte 1 of the same with the
// 8-bit significand.  A flushed value's entry is 0 for either sign.
#ifdef HARAG_GSE_IMAD_ADDR
__device__ __forceinline__ uint32_t mad_hi_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
#endif
__device__ __forceinline__ void enc_gse_sx(const uint4& raw, uint8_t* codes, uint32_t tab, uint32_t e,
                                           uint32_t k11 = 1u << 11, uint32_t k27 = 1u << 27) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t c[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#ifdef HARAG_GSE_IMAD_ADDR
    // entry addresses on the FMA pipe: tab + 4 * (sign|exponent) = mad.hi(w & mask, 2^k, tab)
    // (the multipliers arrive as opaque register values: with literal powers of two ptxas turns the
    // mad.hi back into an ALU shift)
    const uint32_t eh = lds32(mad_hi_u32(w[i] & 0xFF800000u, k11, tab));
    const uint32_t el = lds32(mad_hi_u32(w[i] & 0x0000FF80u, k27, tab));
#else
    const uint32_t eh = lds32(tab | ((w[i] >> 21) & 0x7FCu));
    const uint32_t el = lds32(tab | ((w[i] >> 5) & 0x7FCu));
#endif
    // bits 16..23 = 1.fraction of the high value, 0..7 of the low one, zeros elsewhere: each funnel shift
    // only moves its own value's bits into the byte it reads (3 for high, 1 for low)
    const uint32_t mm = and_or(w[i], 0x00800080u);
    c[2 * i + 1] = eh | __funnelshift_r(0u, mm, eh);
    c[2 * i] = el | __funnelshift_r(0u, mm, el);
  }
  *reinterpret_cast<uint2*>(codes + e) = make_uint2(
      __byte_perm(__byte_perm(c[0], c[1], 0x0071), __byte_perm(c[2], c[3], 0x0071), 0x5410),
      __byte_perm(__byte_perm(c[4], c[5], 0x0071), __byte_perm(c[6], c[7], 0x0071), 0x5410));
}

template <int DT>
__global__ void __cluster_dims__(kGseQ, 1, 1) __launch_bounds__(kGseThreads, HARAG_GSE_MINB)
    gse_slab_kernel(const __grid_constant__ QBatch p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // [code-template table, 2 KB at a 2-KB-aligned address inside the first 4 KB][part | red | bar][source]
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem_raw + ((2048u - (smem_addr(smem_raw) & 2047u)) & 2047u));
  int* part = reinterpret_cast<int*>(smem_raw + 4096);               // [kGseQ][2] quarter ranges (biased)
  int* red = part + 2 * kGseQ;                                       // [warps][2] block reduction
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 4096 + 256);
  uint8_t* src_s = smem_raw + kGseHdr;                               // quarter of the slab's source
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t q = cluster_rank();
  const uint32_t n_slabs = p.L * p.Hl;
  const uint32_t cid = blockIdx.x / kGseQ, j = cid / n_slabs, slab_i = cid - j * n_slabs;
  const uint32_t l = slab_i / p.Hl, hl = slab_i - l * p.Hl;
  const uint32_t qe = p.slab / kGseQ;  // elements per quarter (multiple of 64)
  const QJob& jb = p.jobs[j];
  if (tid == 0) {
    mbar_init(bar, 1);      // the quarter's source (TMA)
    mbar_init(bar + 1, 1);  // the kGseQ quarter ranges (st.async from every CTA of the cluster)
    mbar_arrive_expect_tx(bar + 1, 8 * kGseQ);
    mbar_init_fence();
  }
  __syncthreads();
  // split cluster barrier: every CTA of the cluster must have started before a peer writes into its
  // shared memory (the DSMEM stores below); the wait is placed after the load and the range pass
  cluster_arrive_relaxed();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, 2 * qe);
    bulk_g2s(src_s, jb.src + ((uint64_t)(l * p.H + p.h0 + hl) * p.slab + (uint64_t)q * qe), 2 * qe, bar);
  }
  mbar_wait(bar, 0);
  // quarter range: min / max biased fp32 exponent over nonzero normals (as q_consume_range)
  int emin = 255, emax = 0;
  bool bad = false;
  uint32_t mx = 0u, mn = 0x7FFF7FFFu;  // bf16: running 16-bit-pair max magnitude / min normal key
  for (uint32_t e = tid * 8; e < qe; e += kGseThreads * 8) {
    const uint4 raw = *reinterpret_cast<const uint4*>(src_s + 2 * e);
    if constexpr (DT == HR_BF16) {
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // key = mag + 0x7F80 per half (no carry between the halves: mag <= 0x7FFF): normals (mag >= 0x80)
        // become negative 16-bit values ordered as mag, zeros / subnormals positive, so the signed minimum
        // is the smallest normal whenever the quarter has one
        const uint32_t mag = w[k] & 0x7FFF7FFFu;
        mx = __vmaxu2(mx, mag);
        mn = __vmins2(mn, mag + 0x7F807F80u);
      }
    } else {
      float2 x[4];
      unpack8<DT>(raw, x);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t b = __float_as_uint(k & 1 ? x[k >> 1].y : x[k >> 1].x);
        const int ef = (b >> 23) & 0xFF;
        bad |= ef == 255;
        if (ef != 0) emin = min(emin, ef), emax = max(emax, ef);
      }
    }
  }
  if constexpr (DT == HR_BF16) {
    const uint32_t pmax = max(mx & 0xFFFFu, mx >> 16);
    const int kmin = min((int)(int16_t)(mn & 0xFFFFu), (int)(int16_t)(mn >> 16));
    bad |= pmax >= 0x7F80u;
    emax = (int)(pmax >> 7);
    if (kmin < 0) emin = (int)((((uint32_t)kmin & 0xFFFFu) - 0x7F80u) >> 7);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
    emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
  }
  if (lane == 0) red[2 * warp] = emin, red[2 * warp + 1] = emax;
  __syncthreads();
  cluster_wait();  // every peer CTA is running (pairs with cluster_arrive_relaxed above)
  if (tid == 0) {
    for (uint32_t w = 1; w < kGseThreads / 32; ++w) emin = min(emin, red[2 * w]), emax = max(emax, red[2 * w + 1]);
    // (255 - min, max) as the range pass stores it: a quarter without normals contributes (0, 0)
    const int a = emax != 0 ? 255 - emin : 0, b = emax;
    for (uint32_t r = 0; r < kGseQ; ++r) st_async_cluster_v2(smem_addr(part + 2 * q), smem_addr(bar + 1), r, a, b);
  }
  // every quarter's range is in this CTA's `part` (the peers' stores into this CTA have all landed, so no
  // cluster barrier is needed before exit either)
  mbar_wait(bar + 1, 0);
  int rng[2] = {0, 0};
#pragma unroll
  for (int r = 0; r < kGseQ; ++r) rng[0] = max(rng[0], part[2 * r]), rng[1] = max(rng[1], part[2 * r + 1]);
  const int m = (int)p.gse_m, nmax = 1 << (7 - m);
  const GseArr ga = gse_array(rng, m, nmax);
  // code-template table, indexed by sign|exponent (512 entries; thread t builds exponents t, t + 128, ...
  // and their negative copies).  idx = ceil((E - lo) / step) by a multiply-shift (exact for numerators
  // below 4096 and step 2..4, checked exhaustively offline)
  const uint32_t inv_step = (65536u + (uint32_t)(m - 1) - 1u) / (uint32_t)(m - 1);
  for (int ef = (int)tid; ef < 256; ef += kGseThreads) {
    const int step = m - 1;
    uint32_t ent = 0;
    if (ga.n > 0 && ef >= ga.rmin && ef <= min(ga.rmax, 254)) {
      const int E = ef - 127;
      const int idx = (E <= ga.lo) ? 0 : (int)(((uint32_t)(E - ga.lo + step - 1) * inv_step) >> 16);
      const int d = min(ga.lo + idx * step, ga.Emax) - E;
      if (d <= m - 1) {
        // bf16: sign-free template (the negative half of the table adds the sign); fp16 (enc_gse through
        // fp32, sign combined per element): the "sign kept" bit of gse_build_table
        const uint32_t t7 = (DT == HR_BF16 ? 0u : 0x80u) | ((uint32_t)idx << m);
        ent = (t7 << 24) | (t7 << 8) | (uint32_t)(31 - (m - 1 - d));
      }
    }
    tab[ef] = ent;                                    // positive (and ef = 0: 0)
    tab[256 + ef] = ent ? ent | 0x80008000u : 0u;     // negative: the sign bit rides in the entry
  }
  uint8_t* meta = jb.dst + p.meta_off[HR_S_GSE8] + (uint64_t)slab_i * p.meta_stride[HR_S_GSE8];
  if (q == 0 && warp == 0) gse_write_record(meta, p.meta_stride[HR_S_GSE8], ga, m, nmax, (int)lane);
  __syncthreads();
  uint8_t* codes = jb.dst + (uint64_t)slab_i * p.code_slab[HR_S_GSE8] + (uint64_t)q * qe;
  const uint32_t taddr = smem_addr(tab);
  if constexpr (DT == HR_BF16) {
    for (uint32_t e = tid * 8; e < qe; e += kGseThreads * 8)
      enc_gse_sx(*reinterpret_cast<const uint4*>(src_s + 2 * e), codes, taddr, e, (1u << 11) | (p.n_jobs >> 31),
                 (1u << 27) | (p.n_jobs >> 31));
  } else {  // fp16: through fp32 with the first 256 (sign-free) entries, signs combined per element
    uint32_t nan_acc = 0;
    for (uint32_t e = tid * 8; e < qe; e += kGseThreads * 8)
      enc_gse<DT>(*reinterpret_cast<const uint4*>(src_s + 2 * e), codes, taddr, e, nan_acc);
  }
  if (bad) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------- INT8 / INT4 (G > 256): warp per group
__device__ __forceinline__ void load8(const uint16_t* p, int dt, float (&x)[8]) {
  const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[2 * i] = dt == HR_BF16 ? to_f32<HR_BF16>(w[i] & 0xFFFFu) : to_f32<HR_FP16>(w[i] & 0xFFFFu);
    x[2 * i + 1] = dt == HR_BF16 ? to_f32<HR_BF16>(w[i] >> 16) : to_f32<HR_FP16>(w[i] >> 16);
  }
}
__device__ __forceinline__ bool any_nonfinite(const float (&x)[8]) {
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) bad |= !isfinite(x[i]);
  return bad;
}
// rne(fl(x / s)) for 8 elements (the argument of enc_int4, per element)
__device__ __forceinline__ void div_rne8(const float (&x)[8], float s, int (&q)[8]) {
  float y;
  asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(s));
  const bool slow = !(s >= 1.17549435e-38f && s <= 8.50705917e+37f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float t = __fmul_rn(x[i], y);
    float r = rintf(t);
    if (slow || fabsf(fabsf(__fsub_rn(t, r)) - 0.5f) <= 3.0517578125e-05f) r = rintf(__fdiv_rn(x[i], s));
    q[i] = (int)r;
  }
}

__global__ void __launch_bounds__(256) quant_biggroup_kernel(const __grid_constant__ QBatch p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t slab = p.slab;
  const uint32_t groups_per_slab = (uint32_t)(slab / p.G);
  const uint64_t per_job = (uint64_t)p.L * p.Hl * groups_per_slab;
  const uint64_t n_groups = per_job * p.n_jobs;
  bool bad = false;
  for (uint64_t gi = (blockIdx.x * 256ull + threadIdx.x) / 32; gi < n_groups; gi += (uint64_t)gridDim.x * 8) {
    const uint32_t j = (uint32_t)(gi / per_job);
    const uint64_t gj = gi - j * per_job;
    const QJob& jb = p.jobs[j];
    const uint32_t slab_i = (uint32_t)(gj / groups_per_slab);
    const uint32_t grp = (uint32_t)(gj - (uint64_t)slab_i * groups_per_slab);
    const uint32_t l = slab_i / p.Hl, hl = slab_i - l * p.Hl;
    const uint16_t* src = jb.src + ((uint64_t)l * p.H + p.h0 + hl) * slab;
    uint8_t* codes = jb.dst + slab_i * p.code_slab[jb.scheme];
    uint8_t* meta = jb.dst + p.meta_off[jb.scheme] + (uint64_t)slab_i * p.meta_stride[jb.scheme];
    const uint32_t base = grp * p.G;
    float a = 0.f, mn = INFINITY, mx = -INFINITY;
    for (uint32_t e = base + lane * 8; e < base + p.G; e += kChunk) {  // pass 1: statistics
      float x[8];
      load8(src + e, p.dtype, x);
      bad |= any_nonfinite(x);
#pragma unroll
      for (int i = 0; i < 8; ++i) a = fmaxf(a, fabsf(x[i])), mn = fminf(mn, x[i]), mx = fmaxf(mx, x[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
      mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    float s, m0 = 0.f;
    if (jb.scheme == HR_S_INT8) {
      s = (a == 0.f) ? 1.f : div127(a);
      if (lane == 0) reinterpret_cast<float*>(meta)[grp] = s;
    } else {
      mn = __fadd_rn(mn, 0.f);
      mx = __fadd_rn(mx, 0.f);
      s = (mx == mn) ? 1.f : __fdiv_rn(sub_sat(mx, mn), 15.f);
      m0 = mn;
      if (lane == 0) reinterpret_cast<float2*>(meta)[grp] = make_float2(s, mn);
    }
    for (uint32_t e = base + lane * 8; e < base + p.G; e += kChunk) {  // pass 2: encode (L2 re-read)
      float x[8];
      load8(src + e, p.dtype, x);
      int q[8];
      if (jb.scheme == HR_S_INT8) {
        div_rne8(x, s, q);
        uint32_t w[2] = {0u, 0u};
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i >> 2] |= ((uint32_t)max(-127, min(127, q[i])) & 0xFFu) << (8 * (i & 3));
        *reinterpret_cast<uint2*>(codes + e) = make_uint2(w[0], w[1]);
      } else {
        float u[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) u[i] = sub_sat(x[i], m0);
        div_rne8(u, s, q);
        uint32_t w = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) w |= (uint32_t)max(0, min(15, q[i])) << (4 * i);
        *reinterpret_cast<uint32_t*>(codes + e / 2) = w;
      }
    }
  }
  if (bad) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------- launch
int g_num_sms = 0;

// HARAG_QTILE (tuning only): 0 = every non-GSE scheme on the persistent ring kernel; default 1 = PASS16
// and FP8 on the tile kernel (measured faster: 0.95 / 0.94 of peak vs 0.84 / 0.84), INT8 / INT4 on the
// ring (0.88 / 0.66 vs 0.86 / 0.62)
bool use_tile_kernel() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARAG_QTILE");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
inline bool tile_scheme(uint32_t s) {
#ifdef HARAG_QTILE_GROUPED  // experiment: INT8 / INT4 on the tile kernel too
  if (s == HR_S_INT8 || s == HR_S_INT4) return true;
#endif
  return s == HR_S_PASS16 || s == HR_S_FP8E4M3 || s == HR_S_FP8E5M2 || s == HR_S_MXFP8;
}

template <int DT, int SEG>
void launch_tile(const QBatch& b, cudaStream_t st) {
  const size_t smem = 128 + 2ull * b.tile_e;
  static bool init = false;
  if (!init) {
    HR_CUDA(cudaFuncSetAttribute(quant_tile_kernel<DT, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(128 + 2 * kQTileE)));
    init = true;
  }
  quant_tile_kernel<DT, SEG><<<(unsigned)b.n_tiles, 32 * kTileWarps, smem, st>>>(b);
}

// per-device claim counters of the persistent quantize kernel (64 slots of 16 B, zero between launches;
// slots rotate, so launches on different streams of one device use different counters)
uint32_t* g_qsched[16] = {};
std::atomic<uint32_t> g_qsched_next[16] = {};
std::mutex g_qsched_mu;
const uint64_t g_q_dyn_pct = std::getenv("HARAG_Q_DYN") ? (uint64_t)std::atoi(std::getenv("HARAG_Q_DYN")) : 25;

template <int DT, int SEG, int MODE>
void launch_b(const QBatch& b, cudaStream_t st) {
  if (MODE == MODE_ENCODE && use_tile_kernel()) {
    bool all_tile = b.n_jobs > 0;
    for (uint32_t i = 0; i < b.n_jobs; ++i) all_tile &= tile_scheme(b.jobs[i].scheme);
    if (all_tile) return launch_tile<DT, SEG>(b, st);
  }
  static bool init = false;
  if (!init) {
    HR_CUDA(cudaFuncSetAttribute(quantize_batch_kernel<DT, SEG, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kQSmemBytes));
    init = true;
  }
  const uint64_t grid = std::min<uint64_t>(b.n_tiles, (uint64_t)g_num_sms);
  QBatch bb = b;
  bb.sched = nullptr;
  if (g_q_dyn_pct && b.n_tiles >= 4 * grid) {  // tail balancing (see QBatch::sched)
    int dev = 0;
    HR_CUDA(cudaGetDevice(&dev));
    require(dev < 16, HR_EINVAL, "device index");
    {
      std::lock_guard<std::mutex> g(g_qsched_mu);
      if (!g_qsched[dev]) {
        HR_CUDA(cudaMalloc((void**)&g_qsched[dev], 64 * 16));
        HR_CUDA(cudaMemset(g_qsched[dev], 0, 64 * 16));
      }
    }
    bb.sched = g_qsched[dev] + 4 * (g_qsched_next[dev].fetch_add(1) % 64);
    bb.dyn_tiles = b.n_tiles * g_q_dyn_pct / 100;
    bb.dyn_chunk = (uint32_t)std::max<uint64_t>(1, bb.dyn_tiles / (grid * 8));
  }
  quantize_batch_kernel<DT, SEG, MODE><<<(unsigned)grid, kQThreadsB, kQSmemBytes, st>>>(bb);
}

template <int DT>
void launch_seg(const QBatch& b, int mode, cudaStream_t st) {
  if (mode == MODE_RANGE) return launch_b<DT, 16, MODE_RANGE>(b, st);
  switch (b.G) {  // SEG = G / 8 lanes per group
    case 32: return launch_b<DT, 4, MODE_ENCODE>(b, st);
    case 64: return launch_b<DT, 8, MODE_ENCODE>(b, st);
    case 128: return launch_b<DT, 16, MODE_ENCODE>(b, st);
    case 256: return launch_b<DT, 32, MODE_ENCODE>(b, st);
    default:  // G > 256: the batch holds no INT8 / INT4 job (they take quant_biggroup_kernel)
      require(b.G > 256, HR_EINVAL, "group size must be a power of two >= 32");
      return launch_b<DT, 32, MODE_ENCODE>(b, st);
  }
}

void run_batch(QBatch& b, int mode, cudaStream_t st) {
  bool tile_kernel = mode == MODE_ENCODE && use_tile_kernel() && b.n_jobs > 0;  // as launch_b decides
  for (uint32_t i = 0; i < b.n_jobs; ++i) tile_kernel &= tile_scheme(b.jobs[i].scheme);
  b.tile_e = std::min<uint32_t>(tile_kernel ? kQTileE : kQRingTileE, b.slab);
  b.tiles_per_slab = (b.slab + b.tile_e - 1) / b.tile_e;
  b.n_tiles = (uint64_t)b.n_jobs * b.L * b.Hl * b.tiles_per_slab;
  if (!b.n_tiles) return;
  if (b.dtype == HR_BF16)
    launch_seg<HR_BF16>(b, mode, st);
  else
    launch_seg<HR_FP16>(b, mode, st);
}

}  // namespace

void launch_quantize(const QuantParams* items, int n, cudaStream_t st) {
  if (n <= 0) return;
  if (!g_num_sms) {
    int dev = 0;
    HR_CUDA(cudaGetDevice(&dev));
    HR_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const QuantParams& q0 = items[0];
  const uint64_t slab = (uint64_t)q0.T * q0.D;
  require(slab % kChunk == 0, HR_EINVAL, "T*D must be a multiple of 256");
  require(slab <= (1ull << 31), HR_EINVAL, "slab too large");
  QBatch base{};
  base.L = q0.L, base.H = q0.H, base.Hl = q0.Hl, base.h0 = q0.h0, base.T = q0.T, base.D = q0.D, base.G = q0.G;
  base.g_shift = q0.g_shift, base.gse_e = q0.gse_e, base.gse_m = q0.gse_m, base.dtype = q0.dtype;
  base.slab = (uint32_t)slab;
  base.err = q0.err;
  for (int i = 0; i < n; ++i) {
    const QuantParams& q = items[i];
    require(q.scheme < HR_N_SCHEMES, HR_EINVAL, "unknown scheme");
    require(q.L == q0.L && q.H == q0.H && q.Hl == q0.Hl && q.h0 == q0.h0 && q.T == q0.T && q.D == q0.D &&
                q.G == q0.G && q.dtype == q0.dtype && q.gse_m == q0.gse_m && q.err == q0.err,
            HR_EINVAL, "a quantize batch shares one layout");
    base.code_slab[q.scheme] = q.code_bytes_slab;
    base.meta_off[q.scheme] = q.meta_offset;
    base.meta_stride[q.scheme] = (uint32_t)q.meta_stride;
  }
  const uint64_t n_slabs = (uint64_t)q0.L * q0.Hl;
  // GSE-8 items go in pairs (range pass, then encode while the pair's source is still in L2: a Llama-3-8B
  // K+V pair is 67 MB of the 126 MB L2); every other item of the call shares one encode launch per
  // kQMaxJobs; INT8 / INT4 with G > 256 take the big-group kernel.
  QBatch rng = base, big = base, enc = base, gse = base, tl = base;
  const bool gse_single = 2ull * (slab / kGseQ) <= kGseQMaxBytes && ((slab / kGseQ) % 8) == 0;
  auto flush_gse = [&] {
    if (!gse.n_jobs) return;
    if (gse_single) {  // one pass: a cluster of kGseQ CTAs per slab
      const size_t smem = kGseHdr + 2 * (slab / kGseQ);
      auto kern = gse.dtype == HR_BF16 ? gse_slab_kernel<HR_BF16> : gse_slab_kernel<HR_FP16>;
      static bool init[2] = {false, false};
      if (!init[gse.dtype == HR_BF16]) {
        HR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kGseHdr + kGseQMaxBytes)));
        init[gse.dtype == HR_BF16] = true;
      }
      kern<<<(unsigned)(gse.n_jobs * n_slabs * kGseQ), kGseThreads, smem, st>>>(gse);
      gse.n_jobs = 0;
      return;
    }
    rng.n_jobs = 0;
    for (uint32_t j = 0; j < gse.n_jobs; ++j) {
      HR_CUDA(cudaMemsetAsync(gse.jobs[j].range, 0, sizeof(int) * 2 * n_slabs, st));
      rng.jobs[rng.n_jobs++] = gse.jobs[j];
    }
    run_batch(rng, MODE_RANGE, st);
    run_batch(gse, MODE_ENCODE, st);
    gse.n_jobs = 0;
  };
  auto flush_big = [&] {
    if (!big.n_jobs) return;
    const uint64_t warps = (uint64_t)big.n_jobs * n_slabs * (slab / q0.G);
    const uint64_t grid = std::min<uint64_t>((warps + 7) / 8, (uint64_t)g_num_sms * 8);
    quant_biggroup_kernel<<<(unsigned)grid, 256, 0, st>>>(big);
    big.n_jobs = 0;
  };
  for (int i = 0; i < n; ++i) {
    const QuantParams& q = items[i];
    const QJob job{q.src, q.dst, q.gse_range, q.scheme, 0};
    if (q.scheme == HR_S_GSE8) {
      require(q.gse_range != nullptr, HR_EINVAL, "GSE-8 quantize needs range scratch");
      gse.jobs[gse.n_jobs++] = job;
      if (gse.n_jobs == (gse_single ? (uint32_t)kQMaxJobs : 2u)) flush_gse();
    } else if ((q.scheme == HR_S_INT8 || q.scheme == HR_S_INT4) && q.G > (uint32_t)kChunk) {
      big.jobs[big.n_jobs++] = job;
      if (big.n_jobs == kQMaxJobs) flush_big();
    } else if (use_tile_kernel() && tile_scheme(q.scheme)) {  // elementwise schemes: the tile kernel
      tl.jobs[tl.n_jobs++] = job;
      if (tl.n_jobs == kQMaxJobs) run_batch(tl, MODE_ENCODE, st), tl.n_jobs = 0;
    } else {
      enc.jobs[enc.n_jobs++] = job;
      if (enc.n_jobs == kQMaxJobs) run_batch(enc, MODE_ENCODE, st), enc.n_jobs = 0;
    }
  }
  flush_gse();
  flush_big();
  run_batch(enc, MODE_ENCODE, st);
  run_batch(tl, MODE_ENCODE, st);
  HR_CUDA(cudaGetLastError());
}

}  // namespace harag
