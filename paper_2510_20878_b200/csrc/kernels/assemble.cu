// a8 (+a1) of the HA-RAG hot path on sm_100a: the fused gather -> unpack ->
// dequantise -> scatter of retrieved KV chunks into one contiguous per-request
// KV cache [L][Hl][k*T][D] (north_star), counting item hotness on the way.
//
// Decode rules (oracle: oracle/store.py decode_slab, by the paper's steps):
//   INT8   fl(q * s)                         (R3)
//   INT4   fl(fl(q * s) + mn)                (R4, no FMA)
//   FP8    exact value (cvt.rn.f16x2.e4m3x2 / e5m2x2 are exact)
//   GSE-8  field f != 0:  +-f * 2^(G[idx] - (m-1))   — the marker walk of
//          P:163 written as a denormalised fixed-point number
//   PASS16 bytes unchanged (bulk copy engine both ways)
// then one round-to-nearest-even to the output dtype (R25).
//
// Structure: persistent CTAs, each walking tiles t = blockIdx.x + i*gridDim.x.
// A tile = kAsmTileE consecutive elements of one (request, slot, kind, layer,
// head) slab: its packed codes and the 16-B-aligned window of its group meta
// are fetched by the TMA bulk-copy engine (cp.async.bulk, mbarrier
// complete_tx) into a kAsmStages-deep shared-memory ring, kAsmStages-1 tiles
// ahead; all warps decode from shared memory and write 16-byte vectors, one
// warp instruction covering 512 contiguous output bytes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"

namespace harag {
namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// TMA 1-D bulk copy shared -> global (PASS16 write-back)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void st_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// pack two fp32 into the output dtype with one RNE each
template <int DT>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (DT == HR_BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // cvt.rn.bf16x2.f32, a -> low half
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

// exact int -> float for |v| < 2^22 via the 1.5 * 2^23 magic number
__device__ __forceinline__ float small_int_to_float(int v) {
  return __fsub_rn(__int_as_float(0x4B400000 + v), 12582912.0f);
}
// exact float of the int8 code q in byte `sel` of `word_biased` (= word ^ 0x80808080, i.e. q + 128):
// the float 2^23 + (q + 128) minus (2^23 + 128)
__device__ __forceinline__ float int8_to_float(uint32_t word_biased, uint32_t sel) {
  return __fsub_rn(__uint_as_float(__byte_perm(word_biased, 0x4B000000u, sel)), 8388736.0f);
}

struct TileInfo {
  uint32_t desc, slab_i, sub, l, h, n_el;
};

__device__ __forceinline__ TileInfo tile_info(const AsmParams& p, uint64_t t) {
  const uint64_t per_desc = (uint64_t)p.L * p.Hl * p.tiles_per_slab;
  TileInfo ti;
  ti.desc = (uint32_t)(t / per_desc);
  const uint32_t r = (uint32_t)(t - (uint64_t)ti.desc * per_desc);
  ti.slab_i = r / p.tiles_per_slab;
  ti.sub = r - ti.slab_i * p.tiles_per_slab;
  ti.l = ti.slab_i / p.Hl;
  ti.h = ti.slab_i - ti.l * p.Hl;
  ti.n_el = min((uint32_t)kAsmTileE, p.slab - ti.sub * (uint32_t)kAsmTileE);
  return ti;
}

__device__ __forceinline__ uint32_t code_bytes(uint32_t scheme, uint32_t n_el) {
  return scheme == HR_S_PASS16 ? 2 * n_el : scheme == HR_S_INT4 ? n_el / 2 : n_el;
}
__device__ __forceinline__ uint32_t meta_el(uint32_t scheme) {
  return scheme == HR_S_INT8 ? 4u : scheme == HR_S_INT4 ? 8u : 0u;
}

struct Smem {
  uint8_t codes[kAsmStages][kAsmCodeStage];
  uint8_t meta[kAsmStages][kAsmMetaStage];
  float pow2[kAsmStages][16];
  uint64_t bar[kAsmStages];
};

// Producer (one thread): queue tile t into `stage`.
__device__ __forceinline__ void issue_tile(const AsmParams& p, Smem& sm, uint64_t t, int stage) {
  const TileInfo ti = tile_info(p, t);
  const AsmDesc d = p.descs[ti.desc];
  const uint32_t e0 = ti.sub * (uint32_t)kAsmTileE;
  const uint32_t cb = code_bytes(d.scheme, ti.n_el);
  const uint8_t* csrc = d.codes + (uint64_t)ti.slab_i * code_bytes(d.scheme, p.slab) + code_bytes(d.scheme, e0);
  uint32_t mb = 0;
  const uint8_t* msrc = nullptr;
  if (d.scheme == HR_S_INT8 || d.scheme == HR_S_INT4) {
    const uint32_t me = meta_el(d.scheme);
    const uint32_t g0 = e0 >> p.g_shift, g1 = (e0 + ti.n_el + p.G - 1) >> p.g_shift;
    const uint32_t b0 = (g0 * me) & ~15u, b1 = (g1 * me + 15u) & ~15u;
    msrc = d.meta + (uint64_t)ti.slab_i * p.meta_stride[d.scheme] + b0;
    mb = b1 - b0;
  } else if (d.scheme == HR_S_GSE8) {
    msrc = d.meta + (uint64_t)ti.slab_i * p.meta_stride[d.scheme];
    mb = 16;
  }
  mbar_arrive_expect_tx(&sm.bar[stage], cb + mb);
  bulk_g2s(sm.codes[stage], csrc, cb, &sm.bar[stage]);
  if (mb) bulk_g2s(sm.meta[stage], msrc, mb, &sm.bar[stage]);
}

template <int DT>
__device__ __forceinline__ void decode_int8(const AsmParams& p, const uint8_t* codes, const uint8_t* meta,
                                            uint32_t e0, uint32_t n_el, uint8_t* out) {
  const uint32_t g0 = e0 >> p.g_shift;
  const float* sc = reinterpret_cast<const float*>(meta + ((g0 * 4u) & 15u));
  for (uint32_t e = threadIdx.x * 8; e < n_el; e += kAsmThreads * 8) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    const float s = sc[((e0 + e) >> p.g_shift) - g0];
    const uint32_t u0 = c.x ^ 0x80808080u, u1 = c.y ^ 0x80808080u;  // q + 128
    float f[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[i] = __fmul_rn(int8_to_float(u0, 0x7440u | i), s);
      f[4 + i] = __fmul_rn(int8_to_float(u1, 0x7440u | i), s);
    }
    st_v4(out + 2ull * e, pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]),
          pack2<DT>(f[6], f[7]));
  }
}

template <int DT>
__device__ __forceinline__ void decode_int4(const AsmParams& p, const uint8_t* codes, const uint8_t* meta,
                                            uint32_t e0, uint32_t n_el, uint8_t* out) {
  const uint32_t g0 = e0 >> p.g_shift;
  const float2* sm = reinterpret_cast<const float2*>(meta + ((g0 * 8u) & 15u));
  for (uint32_t e = threadIdx.x * 8; e < n_el; e += kAsmThreads * 8) {
    const uint32_t c = *reinterpret_cast<const uint32_t*>(codes + e / 2);
    const float2 smn = sm[((e0 + e) >> p.g_shift) - g0];
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float q = __fsub_rn(__uint_as_float(0x4B000000u | ((c >> (4 * i)) & 0xFu)), 8388608.0f);
      f[i] = __fadd_rn(__fmul_rn(q, smn.x), smn.y);
    }
    st_v4(out + 2ull * e, pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]),
          pack2<DT>(f[6], f[7]));
  }
}

template <int DT, int SCHEME>
__device__ __forceinline__ void decode_fp8(const uint8_t* codes, uint32_t n_el, uint8_t* out) {
  constexpr __nv_fp8_interpretation_t kInterp = SCHEME == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
  for (uint32_t e = threadIdx.x * 8; e < n_el; e += kAsmThreads * 8) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    const uint32_t w[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)w[i], kInterp);  // exact
      if constexpr (DT == HR_FP16) {
        o[i] = (uint32_t)hr.x | ((uint32_t)hr.y << 16);
      } else {
        const float2 f = __half22float2(*reinterpret_cast<__half2*>(&hr));  // exact
        o[i] = pack2<DT>(f.x, f.y);                                       // exact in bf16
      }
    }
    st_v4(out + 2ull * e, o[0], o[1], o[2], o[3]);
  }
}

template <int DT>
__device__ __forceinline__ void decode_gse(const AsmParams& p, const uint8_t* codes, const float* pow2,
                                           uint32_t n_el, uint8_t* out) {
  const uint32_t m = p.gse_m, fmask = (1u << m) - 1u;
  for (uint32_t e = threadIdx.x * 8; e < n_el; e += kAsmThreads * 8) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t b = ((i < 4 ? c.x : c.y) >> (8 * (i & 3))) & 0xFFu;
      const int fi = (int)(b & fmask);
      const int sf = (b & 0x80u) ? -fi : fi;  // field 0 stays +0
      f[i] = __fmul_rn(small_int_to_float(sf), pow2[(b >> m) & 15u]);
    }
    st_v4(out + 2ull * e, pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]),
          pack2<DT>(f[6], f[7]));
  }
}

template <int DT>
__global__ void __launch_bounds__(kAsmThreads) assemble_kv_kernel(const __grid_constant__ AsmParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  const uint64_t n_my = p.n_tiles > blockIdx.x ? (p.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (tid == 0) {
    for (int s = 0; s < kAsmStages; ++s) mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (uint64_t i = 0; i < n_my && i < (uint64_t)kAsmStages - 1; ++i)
      issue_tile(p, sm, blockIdx.x + i * gridDim.x, (int)i);

  for (uint64_t i = 0; i < n_my; ++i) {
    const int stage = (int)(i % kAsmStages);
    const uint32_t phase = (uint32_t)((i / kAsmStages) & 1);
    if (tid == 0 && i + kAsmStages - 1 < n_my)  // refill the stage drained in iteration i-1
      issue_tile(p, sm, blockIdx.x + (i + kAsmStages - 1) * gridDim.x, (int)((i + kAsmStages - 1) % kAsmStages));

    const uint64_t t = blockIdx.x + i * gridDim.x;
    const TileInfo ti = tile_info(p, t);
    const AsmDesc d = p.descs[ti.desc];
    const uint32_t e0 = ti.sub * (uint32_t)kAsmTileE;
    uint8_t* out = d.out + 2ull * (((uint64_t)ti.slab_i * p.k + d.slot) * p.slab + e0);
    if (tid == 0 && d.count != nullptr && ti.slab_i == 0 && ti.sub == 0) atomicAdd(d.count, 1ull);  // a1

    mbar_wait(&sm.bar[stage], phase);
    const uint8_t* codes = sm.codes[stage];
    switch (d.scheme) {
      case HR_S_PASS16:
        if (tid == 0) {
          bulk_s2g(out, codes, 2 * ti.n_el);
          bulk_wait_read_all();  // smem stage may be refilled after the barrier below
        }
        break;
      case HR_S_INT8:
        decode_int8<DT>(p, codes, sm.meta[stage], e0, ti.n_el, out);
        break;
      case HR_S_INT4:
        decode_int4<DT>(p, codes, sm.meta[stage], e0, ti.n_el, out);
        break;
      case HR_S_FP8E4M3:
        decode_fp8<DT, HR_S_FP8E4M3>(codes, ti.n_el, out);
        break;
      case HR_S_FP8E5M2:
        decode_fp8<DT, HR_S_FP8E5M2>(codes, ti.n_el, out);
        break;
      case HR_S_GSE8: {
        float* pow2 = sm.pow2[stage];
        if (tid < 16) {  // 2^(G_i - (m-1)), exact (fp32 subnormal below 2^-126)
          const int k = (int)(int8_t)sm.meta[stage][tid] - ((int)p.gse_m - 1);
          pow2[tid] = k >= -126 ? __int_as_float((k + 127) << 23) : (k >= -149 ? __int_as_float(1 << (k + 149)) : 0.f);
        }
        __syncthreads();
        decode_gse<DT>(p, codes, pow2, ti.n_el, out);
        break;
      }
      default:
        break;
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait_all();
}

int g_ctas_per_sm = 0;
int g_num_sms = 0;

template <int DT>
void setup_kernel() {
  HR_CUDA(cudaFuncSetAttribute(assemble_kv_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sizeof(Smem)));
}

}  // namespace

int assemble_ctas_per_sm() {
  if (!g_ctas_per_sm) {
    setup_kernel<HR_BF16>();
    setup_kernel<HR_FP16>();
    HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_ctas_per_sm, assemble_kv_kernel<HR_BF16>, kAsmThreads,
                                                          sizeof(Smem)));
    int dev = 0;
    HR_CUDA(cudaGetDevice(&dev));
    HR_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    if (g_ctas_per_sm < 1) g_ctas_per_sm = 1;
  }
  return g_ctas_per_sm;
}

void launch_assemble(const AsmParams& p, cudaStream_t st, int grid_ctas) {
  if (p.n_tiles == 0) return;
  const int per_sm = assemble_ctas_per_sm();
  uint64_t grid = grid_ctas > 0 ? (uint64_t)grid_ctas : (uint64_t)g_num_sms * per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  if (p.dtype == HR_BF16)
    assemble_kv_kernel<HR_BF16><<<(unsigned)grid, kAsmThreads, sizeof(Smem), st>>>(p);
  else
    assemble_kv_kernel<HR_FP16><<<(unsigned)grid, kAsmThreads, sizeof(Smem), st>>>(p);
  HR_CUDA(cudaGetLastError());
}

}  // namespace harag
