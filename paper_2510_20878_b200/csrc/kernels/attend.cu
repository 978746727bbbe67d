// Consumer of the assembled KV: attention of a request's
// query rows over its retrieved chunks, reading the PACKED codes of the store
// directly — gather + unpack + dequantise fused into the attention kernel, so
// the 2 B/element KV cache of hr_assemble_kv is never written to HBM.
//
//   O[r][l][hq][i] = sum_j softmax_j(scale * <q_i, k_j>) v_j,   LSE = log sum_j exp(scale * <q_i, k_j>)
//
// over the k*T keys of request r (docs in request order), GQA: query head hq
// reads KV head hq / g.  This is the cross-attention of the question tokens
// to the precomputed chunk KV that TurboRAG / HA-RAG prefill performs (P:41,
// P:316); LSE lets a caller merge it with the question's own causal part.
//
// sm_100a design: one CTA per (request, layer, KV head) unit; the unit's
// M = g*n_q query rows (<= 128) form the A operand of tcgen05.mma (M = 128,
// rows past M are zero).  Per 64-key tile: all threads decode the K and V
// codes straight from HBM into bf16/fp16 operand tiles in shared memory
// (the decode of hr_assemble_kv, bit for bit); one thread issues S = Q K^T
// into TMEM; each thread owns one query row for the online softmax (tcgen05.ld
// of its S row, exp2, lazy rescale of O only when the running max grows by
// more than 2^8), writes P to shared memory; one thread issues O += P V into
// TMEM.  Operand tiles use the canonical no-swizzle core-matrix layouts
// (8 rows x 16 B per core matrix).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"

namespace harag {
namespace {

constexpr int kAttThreads = 128;  // 4 warps: thread t owns query row t (TMEM lane t)
constexpr int kKT = 64;           // keys per tile
constexpr int kRows = 128;        // MMA M

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, no swizzle (canonical core-matrix layout): start address,
// LBO = byte distance between core matrices adjacent in K, SBO = adjacent in M/N; version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Instruction descriptor, kind::f16: fp32 accumulate, A/B format (0 fp16, 1 bf16), majors, N, M.
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, uint32_t a_mn, uint32_t b_mn, uint32_t n, uint32_t m) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
               : "memory");
}

#define HR_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), \
                 "=r"(v[i + 6]), "=r"(v[i + 7])
#define HR_W8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), \
                 "r"(v[i + 6]), "r"(v[i + 7])
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : HR_R8(0), HR_R8(8), HR_R8(16), HR_R8(24)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      HR_W8(0), HR_W8(8), HR_W8(16), HR_W8(24)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
#undef HR_R8
#undef HR_W8

template <int DT>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (DT == HR_BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}
template <int DT>
__device__ __forceinline__ float lo_f(uint32_t w) {
  return DT == HR_BF16 ? __uint_as_float(w << 16) : __half2float(__ushort_as_half((unsigned short)(w & 0xFFFFu)));
}
template <int DT>
__device__ __forceinline__ float hi_f(uint32_t w) {
  return DT == HR_BF16 ? __uint_as_float(w & 0xFFFF0000u) : __half2float(__ushort_as_half((unsigned short)(w >> 16)));
}
__device__ __forceinline__ float s8f(uint32_t w, int byte) { return (float)(int8_t)(w >> (8 * byte)); }
__device__ __forceinline__ float u8f(uint32_t w, int byte) { return (float)(uint8_t)(w >> (8 * byte)); }

// Decode the 8 elements [e, e+8) of one slab — the decode rules of hr_assemble_kv (R3-R5, R9) bit for bit.
template <int DT>
__device__ __forceinline__ uint4 decode8(uint32_t scheme, const uint8_t* codes, const uint8_t* meta, uint32_t e,
                                         uint32_t g_shift, uint32_t gse_m, const float* gtab) {
  switch (scheme) {
    case HR_S_PASS16:
      return __ldg(reinterpret_cast<const uint4*>(codes + 2ull * e));
    case HR_S_INT8: {
      const uint2 c = __ldg(reinterpret_cast<const uint2*>(codes + e));
      const float s = __ldg(reinterpret_cast<const float*>(meta) + (e >> g_shift));
      return make_uint4(pack2<DT>(__fmul_rn(s8f(c.x, 0), s), __fmul_rn(s8f(c.x, 1), s)),
                        pack2<DT>(__fmul_rn(s8f(c.x, 2), s), __fmul_rn(s8f(c.x, 3), s)),
                        pack2<DT>(__fmul_rn(s8f(c.y, 0), s), __fmul_rn(s8f(c.y, 1), s)),
                        pack2<DT>(__fmul_rn(s8f(c.y, 2), s), __fmul_rn(s8f(c.y, 3), s)));
    }
    case HR_S_INT4: {
      const uint32_t c = __ldg(reinterpret_cast<const uint32_t*>(codes + e / 2));
      const uint32_t lo = c & 0x0F0F0F0Fu, hi = (c >> 4) & 0x0F0F0F0Fu;
      const float2 q = __ldg(reinterpret_cast<const float2*>(meta) + (e >> g_shift));
      float f[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        f[2 * i] = __fadd_rn(__fmul_rn(u8f(lo, i), q.x), q.y);
        f[2 * i + 1] = __fadd_rn(__fmul_rn(u8f(hi, i), q.x), q.y);
      }
      return make_uint4(pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]), pack2<DT>(f[6], f[7]));
    }
    case HR_S_FP8E4M3:
    case HR_S_FP8E5M2: {
      const __nv_fp8_interpretation_t it = scheme == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
      const uint2 c = __ldg(reinterpret_cast<const uint2*>(codes + e));
      const uint32_t w[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)w[i], it);  // exact
        if constexpr (DT == HR_FP16) {
          o[i] = (uint32_t)hr.x | ((uint32_t)hr.y << 16);
        } else {
          const float2 f = __half22float2(*reinterpret_cast<__half2*>(&hr));
          o[i] = pack2<DT>(f.x, f.y);  // exact in bf16
        }
      }
      return make_uint4(o[0], o[1], o[2], o[3]);
    }
    default: {  // GSE-8: +-f * 2^(G_idx - (m-1)) from the slab's fp32 table (staged in shared memory)
      const uint2 c = __ldg(reinterpret_cast<const uint2*>(codes + e));
      const uint32_t fm = (1u << gse_m) - 1u;
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t b = ((i < 4 ? c.x : c.y) >> (8 * (i & 3))) & 0xFFu;
        f[i] = __fmaf_rn((float)(b & fm), gtab[b >> gse_m], 0.f);
      }
      return make_uint4(pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]), pack2<DT>(f[6], f[7]));
    }
  }
}

struct AttSmem {
  uint8_t* q;  // [128 rows][D] K-major core layout: (dc * 16 + row / 8) * 128 + (row % 8) * 16
  uint8_t* k;  // [64 keys][D]  K-major (B of S = Q K^T)
  uint8_t* v;  // [64 keys][D]  MN-major (B of O += P V): (key / 8 * (D / 8) + dc) * 128 + (key % 8) * 16
  uint8_t* p;  // [128 rows][64 keys] K-major (A of O += P V)
  float* gtab; // [2][32] GSE decode tables of the current K and V slab
  uint64_t* bar;  // [2]: S done, O done
  uint32_t* tmem; // TMEM base written by tcgen05.alloc
};

size_t att_smem_bytes(uint32_t D) {
  return (size_t)kRows * D * 2 + 2 * (size_t)kKT * D * 2 + (size_t)kRows * kKT * 2 + 2 * 32 * 4 + 2 * 8 + 16;
}

template <int DT>
__global__ void __launch_bounds__(kAttThreads) attend_kernel(AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t D = p.D;
  AttSmem sm;
  sm.q = smem_raw;
  sm.k = sm.q + kRows * D * 2;
  sm.v = sm.k + kKT * D * 2;
  sm.p = sm.v + kKT * D * 2;
  sm.gtab = reinterpret_cast<float*>(sm.p + kRows * kKT * 2);
  sm.bar = reinterpret_cast<uint64_t*>(sm.gtab + 64);
  sm.tmem = reinterpret_cast<uint32_t*>(sm.bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;

  const uint32_t unit = blockIdx.x;  // (request, layer, head)
  const uint32_t r = unit / (p.L * p.Hl), lh = unit - r * (p.L * p.Hl);
  const uint32_t l = lh / p.Hl, h = lh - l * p.Hl;
  const uint32_t slab_i = l * p.Hl + h;
  const uint32_t hq = p.Hl * p.g;  // query heads on this rank
  const uint64_t row0 = (((uint64_t)r * p.L + l) * hq + (uint64_t)h * p.g) * p.n_q;  // first query row of the unit

  if (warp == 0) {  // TMEM: S at columns [0, 64), O at [128, 128 + D)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(sm.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (p.descs[0].count != nullptr && l == 0 && h == 0) {  // a1: hotness of this request's items
      for (uint32_t j = 0; j < 2 * p.k; ++j) {
        const AsmDesc& d = p.descs[(uint64_t)r * 2 * p.k + j];
        if (d.count) atomicAdd(d.count, 1ull);
      }
    }
  }
  // Q tile: rows >= M are zero.  Thread mapping per 32 chunks: 8 rows x 4 column chunks (coalesced
  // 64-B row reads, conflict-free 16-B shared stores).
  const uint32_t dcs = D / 8;
  for (uint32_t c = tid; c < kRows * dcs; c += kAttThreads) {
    const uint32_t gI = c >> 5, i = c & 7, jj = (c >> 3) & 3;
    const uint32_t row = (gI % (kRows / 8)) * 8 + i, dc = (gI / (kRows / 8)) * 4 + jj;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < p.M) v = __ldg(reinterpret_cast<const uint4*>(p.q + (row0 + row) * D) + dc);
    *reinterpret_cast<uint4*>(sm.q + (dc * (kRows / 8) + row / 8) * 128 + (row % 8) * 16) = v;
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *sm.tmem;
  const uint32_t t_s = tmem, t_o = tmem + 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;

  const uint32_t fmt = DT == HR_BF16 ? 1u : 0u;
  const uint32_t id_s = idesc(fmt, 0, 0, kKT, kRows);  // S[128 x 64] = Q[128 x D] . K[64 x D]^T
  const uint32_t id_o = idesc(fmt, 0, 1, D, kRows);    // O[128 x D] += P[128 x 64] . V[64 x D] (V MN-major)
  const uint32_t tiles_per_doc = p.T / kKT;
  const uint32_t n_tiles = p.k * tiles_per_doc;
  const float c = p.scale_log2;
  float m_ref = -INFINITY, lsum = 0.f;

  for (uint32_t j = 0; j < n_tiles; ++j) {
    const uint32_t slot = j / tiles_per_doc, t0 = (j - slot * tiles_per_doc) * kKT;
    const AsmDesc& dk = p.descs[((uint64_t)r * p.k + slot) * 2];
    const AsmDesc& dv = p.descs[((uint64_t)r * p.k + slot) * 2 + 1];
    const uint8_t* kc = dk.codes + (uint64_t)slab_i * p.code_slab[dk.scheme];
    const uint8_t* vc = dv.codes + (uint64_t)slab_i * p.code_slab[dv.scheme];
    const uint8_t* km = dk.meta + (uint64_t)slab_i * p.meta_stride[dk.scheme];
    const uint8_t* vm = dv.meta + (uint64_t)slab_i * p.meta_stride[dv.scheme];
    if (t0 == 0) {  // new doc: stage the GSE decode tables of its K and V slab
      __syncthreads();
      if (tid < 64) {
        const bool isv = tid >= 32;
        const AsmDesc& d = isv ? dv : dk;
        const uint8_t* m = isv ? vm : km;
        const uint32_t i = tid & 31;
        sm.gtab[tid] = (d.scheme == HR_S_GSE8 && i < (2u << p.gse_e)) ? reinterpret_cast<const float*>(m + 16)[i] : 0.f;
      }
      __syncthreads();
    }
    // decode the K and V tiles (64 keys x D) into the operand layouts
    for (uint32_t cc = tid; cc < kKT * dcs; cc += kAttThreads) {
      const uint32_t gI = cc >> 5, i = cc & 7, jj = (cc >> 3) & 3;
      const uint32_t key = (gI % (kKT / 8)) * 8 + i, dc = (gI / (kKT / 8)) * 4 + jj;
      const uint32_t e = (t0 + key) * D + dc * 8;
      const uint4 kv = decode8<DT>(dk.scheme, kc, km, e, p.g_shift, p.gse_m, sm.gtab);
      const uint4 vv = decode8<DT>(dv.scheme, vc, vm, e, p.g_shift, p.gse_m, sm.gtab + 32);
      *reinterpret_cast<uint4*>(sm.k + (dc * (kKT / 8) + key / 8) * 128 + (key % 8) * 16) = kv;
      *reinterpret_cast<uint4*>(sm.v + ((key / 8) * dcs + dc) * 128 + (key % 8) * 16) = vv;
      if (p.kv_dump) {  // test hook: the assembled KV [r][2][l][h][k*T][D]
        const uint64_t base = ((((uint64_t)r * 2) * p.L + l) * p.Hl + h) * p.k * p.T * D;
        const uint64_t kvoff = (uint64_t)p.L * p.Hl * p.k * p.T * D;
        const uint64_t o = base + ((uint64_t)slot * p.T + t0 + key) * D + dc * 8;
        *reinterpret_cast<uint4*>(p.kv_dump + o) = kv;
        *reinterpret_cast<uint4*>(p.kv_dump + kvoff + o) = vv;
      }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (tid == 0) {
      tc_after();
      const uint32_t qa = saddr(sm.q), ka = saddr(sm.k);
      for (uint32_t s = 0; s < D / 16; ++s)  // K-major: one k-step = 2 core matrices along K
        mma_f16(t_s, sdesc(qa + s * 2 * (kRows / 8) * 128, (kRows / 8) * 128, 128),
                sdesc(ka + s * 2 * (kKT / 8) * 128, (kKT / 8) * 128, 128), id_s, s > 0);
      mma_commit(&sm.bar[0]);
    }
    mbar_wait(&sm.bar[0], j & 1);
    tc_after();
    // online softmax on this thread's row
    uint32_t sv[2][32];
    tmem_ld32(t_s + lane_base, sv[0]);
    tmem_ld32(t_s + lane_base + 32, sv[1]);
    float mt = -INFINITY;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 32; ++b) mt = fmaxf(mt, __uint_as_float(sv[a][b]) * c);
    const bool grow = mt > m_ref + 8.f;  // lazy rescale: p stays <= 2^8 between rescales
    const float m_new = grow ? mt : m_ref;
    if (__any_sync(0xFFFFFFFFu, grow) && j > 0) {
      const float alpha = grow ? exp2f(m_ref - m_new) : 1.f;
      for (uint32_t cb = 0; cb < D; cb += 32) {
        uint32_t ov[32];
        tmem_ld32(t_o + lane_base + cb, ov);
#pragma unroll
        for (int b = 0; b < 32; ++b) ov[b] = __float_as_uint(__uint_as_float(ov[b]) * alpha);
        tmem_st32(t_o + lane_base + cb, ov);
      }
      lsum *= alpha;
    }
    m_ref = m_new;
    uint8_t* prow = sm.p + (tid / 8) * 128 + (tid % 8) * 16;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // 8 keys -> one 16-B core-matrix row
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float p0 = exp2f(__uint_as_float(sv[a][q * 8 + 2 * u]) * c - m_ref);
          const float p1 = exp2f(__uint_as_float(sv[a][q * 8 + 2 * u + 1]) * c - m_ref);
          w[u] = pack2<DT>(p0, p1);
          lsum += lo_f<DT>(w[u]) + hi_f<DT>(w[u]);  // normalise by the rounded weights actually used
        }
        const uint32_t kc8 = a * 4 + q;  // key chunk
        *reinterpret_cast<uint4*>(prow + kc8 * (kRows / 8) * 128) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (tid == 0) {
      tc_after();
      const uint32_t pa = saddr(sm.p), va = saddr(sm.v);
      for (uint32_t s = 0; s < kKT / 16; ++s)
        mma_f16(t_o, sdesc(pa + s * 2 * (kRows / 8) * 128, (kRows / 8) * 128, 128),
                sdesc(va + s * 2 * dcs * 128, dcs * 128, 128), id_o, (j > 0 || s > 0) ? 1u : 0u);
      mma_commit(&sm.bar[1]);
    }
    mbar_wait(&sm.bar[1], j & 1);
    tc_after();
  }
  // epilogue: O / l -> output dtype; LSE (natural log) = ln 2 * (m_ref + log2 l)
  const float inv = 1.f / lsum;
  for (uint32_t cb = 0; cb < D; cb += 32) {
    uint32_t ov[32];
    tmem_ld32(t_o + lane_base + cb, ov);
    if ((uint32_t)tid < p.M) {
      uint4* dst = reinterpret_cast<uint4*>(p.o + (row0 + tid) * D + cb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          w[u] = pack2<DT>(__uint_as_float(ov[q * 8 + 2 * u]) * inv, __uint_as_float(ov[q * 8 + 2 * u + 1]) * inv);
        dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  if ((uint32_t)tid < p.M && p.lse) p.lse[row0 + tid] = 0.69314718055994531f * (m_ref + __log2f(lsum));
  tc_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

}  // namespace

void launch_attend(const AttnParams& p, cudaStream_t st) {
  require(p.D == 64 || p.D == 128, HR_EINVAL, "attend: head_dim must be 64 or 128");
  require(p.T % kKT == 0, HR_EINVAL, "attend: tokens per chunk must be a multiple of 64");
  require(p.M >= 1 && p.M <= kRows, HR_EINVAL, "attend: g * n_q must be in [1, 128]");
  const size_t smem = att_smem_bytes(p.D);
  const uint64_t units = (uint64_t)p.n_req * p.L * p.Hl;
  if (!units) return;
  require(units < (1ull << 31), HR_EINVAL, "attend: too many units");
  if (p.dtype == HR_BF16) {
    static bool init = false;
    if (!init) {
      HR_CUDA(cudaFuncSetAttribute(attend_kernel<HR_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)att_smem_bytes(128)));
      init = true;
    }
    attend_kernel<HR_BF16><<<(unsigned)units, kAttThreads, smem, st>>>(p);
  } else {
    static bool init = false;
    if (!init) {
      HR_CUDA(cudaFuncSetAttribute(attend_kernel<HR_FP16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)att_smem_bytes(128)));
      init = true;
    }
    attend_kernel<HR_FP16><<<(unsigned)units, kAttThreads, smem, st>>>(p);
  }
  HR_CUDA(cudaGetLastError());
}

}  // namespace harag
