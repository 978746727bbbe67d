// a8 (+a1) of the HA-RAG hot path on sm_100a: the fused gather -> unpack ->
// dequantise -> scatter of retrieved KV chunks into one contiguous per-request
// KV cache [L][Hl][k*T][D] (north_star), counting item hotness on the way.
//
// Decode rules (oracle: oracle/store.py decode_slab, which follows the paper's steps):
//   INT8   fl(q * s)                         (R3)
//   INT4   fl(fl(q * s) + mn)                (R4, no FMA)
//   FP8    exact value (cvt.rn.f16x2.e4m3x2 / e5m2x2 are exact)
//   GSE-8  field f != 0:  +-f * 2^(G[idx] - (m-1)), field 0: +0 — the marker
//          walk of P:163 written as a denormalised fixed-point number
//          (identity proven in tests/test_oracle_codecs.py::test_gse_decode_closed_form)
//   PASS16 bytes unchanged (TMA bulk copy both ways)
// then one round-to-nearest-even to the output dtype (R25).
//
// Structure (warp-specialised, persistent): CTA = 1 producer warp + 28
// consumer warps (HARAG_CONSUMER_WARPS, kernels.h; one CTA per SM); CTA b owns
// a contiguous block of tiles.  A tile = p.tile_e
// consecutive elements of one (request, slot, kind, layer, head) slab.  The
// producer lane resolves the tile (descriptor, addresses, hotness count),
// writes a small header to shared memory and has the TMA engine bulk-copy
// the tile's packed codes and the 16-B-aligned window of its group meta into
// a kAsmStages-deep ring (mbarrier "full", complete_tx).  Consumer warps
// decode from shared memory and write 16-byte vectors (one warp instruction
// = 512 contiguous output bytes), then release the stage on mbarrier "empty".
// No CTA-wide barrier in the loop.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "../common.h"
#include "../kernels.h"

#include <algorithm>

namespace harag {
namespace {

constexpr int kConsumerWarps = kAsmThreads / 32 - 1;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
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
#ifdef HARAG_ST_CS
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
#else
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
#endif
}

// two fp32 -> output dtype, one RNE each (first argument -> low half)
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

// byte `byte` of w as an exact float (I2F.S8 / I2F.U8 with a byte selector)
__device__ __forceinline__ float s8f(uint32_t w, int byte) { return (float)(int8_t)(w >> (8 * byte)); }
__device__ __forceinline__ float u8f(uint32_t w, int byte) { return (float)(uint8_t)(w >> (8 * byte)); }

__device__ __forceinline__ uint32_t code_bytes(uint32_t scheme, uint32_t n_el) {
  return scheme == HR_S_PASS16 ? 2 * n_el : scheme == HR_S_INT4 ? n_el / 2 : n_el;
}

struct TileHdr {
  uint8_t* out;      // first output byte of the tile
  uint32_t n_el;     // elements in the tile (ragged last tile of a slab)
  uint32_t scheme;
  uint32_t meta_off; // byte offset of the tile's first group inside the meta window
  uint32_t goff;     // e0 mod G: group of element e is (goff + e) >> g_shift
};

// Descriptors: launches of <= kAsmInline (64) descriptors (a single request, a streamed item) carry
// them in the kernel parameters (p.descs == nullptr), larger ones read a device array.
//
// Dynamic shared memory: [codes ring | meta ring | headers | full barriers | empty barriers];
// every meta stage starts 256-B aligned
struct Smem {
  uint8_t* base;
  uint32_t meta_stage;
  __device__ __forceinline__ uint8_t* codes(int s) const { return base + s * kAsmCodeStage; }
  __device__ __forceinline__ uint8_t* meta(int s) const {
    return base + kAsmStages * kAsmCodeStage + s * meta_stage;
  }
  __device__ __forceinline__ TileHdr* hdr() const {
    return reinterpret_cast<TileHdr*>(base + kAsmStages * (kAsmCodeStage + meta_stage));
  }
  __device__ __forceinline__ uint64_t* full() const { return reinterpret_cast<uint64_t*>(hdr() + kAsmStages); }
  __device__ __forceinline__ uint64_t* empty() const { return full() + kAsmStages; }
};

size_t smem_bytes(uint32_t meta_stage) {
  return (size_t)kAsmStages * (kAsmCodeStage + meta_stage) + kAsmStages * sizeof(TileHdr) + 2 * kAsmStages * 8;
}

// Blocked distribution of the first n_tiles - dyn_tiles tiles: CTA b owns [b*n/grid, (b+1)*n/grid) —
// consecutive tiles of one slab / item, so the producer reloads a descriptor only when it crosses an item.
// The last dyn_tiles are claimed in chunks through p.sched (the CTAs that finish their block first take
// more of them: the static split left the slowest CTA ~5% behind on a single request).
__device__ __forceinline__ void my_tiles(const AsmParams& p, uint64_t& t0, uint64_t& t1) {
  const uint64_t ns = p.sched ? p.n_tiles - p.dyn_tiles : p.n_tiles;
  t0 = ns * blockIdx.x / gridDim.x;
  t1 = ns * (blockIdx.x + 1) / gridDim.x;
}

// ------------------------------------------------------------------ producer
__device__ __forceinline__ void produce(const AsmParams& p, const Smem& sm) {
  const uint32_t per_desc = p.L * p.Hl * p.tiles_per_slab;
  const uint32_t n_slabs = p.L * p.Hl;
  uint64_t i = 0;  // stage sequence number across every range this CTA produces
  auto range = [&](uint64_t t0, uint64_t t1) {
    if (t1 <= t0) return;
    uint32_t di = (uint32_t)(t0 / per_desc);
    uint32_t r = (uint32_t)(t0 - (uint64_t)di * per_desc);
    uint32_t slab_i = r / p.tiles_per_slab;
    uint32_t sub = r - slab_i * p.tiles_per_slab;
    AsmDesc d = p.descs ? p.descs[di] : p.inl[di];
    for (uint64_t t = t0; t < t1; ++t, ++i) {
      const int stage = (int)(i % kAsmStages);
      if (i >= kAsmStages) mbar_wait(&sm.empty()[stage], (uint32_t)(((i / kAsmStages) - 1) & 1));
      const uint32_t e0 = sub * p.tile_e;
      const uint32_t n_el = min(p.tile_e, p.slab - e0);
      const uint32_t cb = code_bytes(d.scheme, n_el);
      const uint8_t* csrc = d.codes + (uint64_t)slab_i * code_bytes(d.scheme, p.slab) + code_bytes(d.scheme, e0);
      uint32_t mb = 0, moff = 0;
      const uint8_t* msrc = nullptr;
      if (d.scheme == HR_S_INT8 || d.scheme == HR_S_INT4 || d.scheme == HR_S_MXFP8) {
        // the tile's window of group records: INT8 fp32 s, INT4 (s, mn) per group of G; MXFP8 one E8M0
        // byte per 32 elements
        const bool mx = d.scheme == HR_S_MXFP8;
        const uint32_t me = d.scheme == HR_S_INT8 ? 4u : mx ? 1u : 8u, gs = mx ? 5u : p.g_shift;
        const uint32_t g0 = e0 >> gs, g1 = (e0 + n_el + (1u << gs) - 1) >> gs;
        const uint32_t b0 = (g0 * me) & ~15u, b1 = (g1 * me + 15u) & ~15u;
        msrc = d.meta + (uint64_t)slab_i * p.meta_stride[d.scheme] + b0;
        mb = b1 - b0;
        moff = g0 * me - b0;
      } else if (d.scheme == HR_S_GSE8) {  // whole record: shared-exponent array + fp32 decode table
        msrc = d.meta + (uint64_t)slab_i * p.meta_stride[d.scheme];
        mb = p.meta_stride[d.scheme];
      }
      TileHdr& h = sm.hdr()[stage];
      h.out = d.out + 2ull * (((uint64_t)slab_i * p.k + d.slot) * p.slab + e0);
      h.n_el = n_el;
      h.scheme = d.scheme;
      h.meta_off = moff;
      h.goff = e0 & (p.G - 1);
      if (d.count != nullptr && slab_i == 0 && sub == 0) atomicAdd(d.count, 1ull);  // a1
      uint64_t* full = &sm.full()[stage];
      mbar_arrive_expect_tx(full, cb + mb);  // release: the header is visible with the phase flip
      bulk_g2s(sm.codes(stage), csrc, cb, full);
      if (mb) bulk_g2s(sm.meta(stage), msrc, mb, full);
      if (++sub == p.tiles_per_slab) {  // advance (sub, slab, descriptor) without divisions
        sub = 0;
        if (++slab_i == n_slabs) {
          slab_i = 0;
          if (t + 1 < t1) {
            ++di;
            d = p.descs ? p.descs[di] : p.inl[di];
          }
        }
      }
    }
  };
  uint64_t t0, t1;
  my_tiles(p, t0, t1);
  range(t0, t1);
  if (p.sched) {
    const uint64_t base = p.n_tiles - p.dyn_tiles;
    while (true) {
      const uint64_t c = atomicAdd(reinterpret_cast<unsigned long long*>(p.sched), (unsigned long long)p.dyn_chunk);
      if (c >= p.dyn_tiles) break;
      range(base + c, base + min(c + p.dyn_chunk, p.dyn_tiles));
    }
    // end of this CTA's tiles: a header with n_el = 0 in the next stage
    const int stage = (int)(i % kAsmStages);
    if (i >= kAsmStages) mbar_wait(&sm.empty()[stage], (uint32_t)(((i / kAsmStages) - 1) & 1));
    sm.hdr()[stage].n_el = 0;
    mbar_arrive(&sm.full()[stage]);
    // the last producer to finish claiming resets the counter for the next launch on the stream
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned int*>(p.sched) + 2, 1u) == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned long long*>(p.sched) = 0ull;
      reinterpret_cast<volatile unsigned int*>(p.sched)[2] = 0u;
    }
  }
}

// ------------------------------------------------------------------ consumers
// Consumer thread ctid handles the 8-element chunks ctid, ctid + 32*kConsumerWarps, ... of a tile.
constexpr uint32_t kChunkStride = kConsumerWarps * 32 * 8;

template <int DT>
__device__ __forceinline__ void decode_int8(const TileHdr& h, const uint8_t* codes, const uint8_t* meta, int ctid,
                                            uint32_t g_shift) {
  const float* sc = reinterpret_cast<const float*>(meta + h.meta_off);
#pragma unroll 2
  for (uint32_t e = ctid * 8; e < h.n_el; e += kChunkStride) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    const float s = sc[(h.goff + e) >> g_shift];
    st_v4(h.out + 2ull * e, pack2<DT>(__fmul_rn(s8f(c.x, 0), s), __fmul_rn(s8f(c.x, 1), s)),
          pack2<DT>(__fmul_rn(s8f(c.x, 2), s), __fmul_rn(s8f(c.x, 3), s)),
          pack2<DT>(__fmul_rn(s8f(c.y, 0), s), __fmul_rn(s8f(c.y, 1), s)),
          pack2<DT>(__fmul_rn(s8f(c.y, 2), s), __fmul_rn(s8f(c.y, 3), s)));
  }
}

template <int DT>
__device__ __forceinline__ void decode_int4(const TileHdr& h, const uint8_t* codes, const uint8_t* meta, int ctid,
                                            uint32_t g_shift) {
  const float2* sm = reinterpret_cast<const float2*>(meta + h.meta_off);
#pragma unroll 2
  for (uint32_t e = ctid * 8; e < h.n_el; e += kChunkStride) {
    const uint32_t c = *reinterpret_cast<const uint32_t*>(codes + e / 2);
    const uint32_t lo = c & 0x0F0F0F0Fu, hi = (c >> 4) & 0x0F0F0F0Fu;  // even / odd elements
    const float2 q = sm[(h.goff + e) >> g_shift];                       // (s, mn)
    float f[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __fadd_rn(__fmul_rn(u8f(lo, i), q.x), q.y);
      f[2 * i + 1] = __fadd_rn(__fmul_rn(u8f(hi, i), q.x), q.y);
    }
    st_v4(h.out + 2ull * e, pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]),
          pack2<DT>(f[6], f[7]));
  }
}

template <int DT, int SCHEME>
__device__ __forceinline__ void decode_fp8(const TileHdr& h, const uint8_t* codes, int ctid) {
  constexpr __nv_fp8_interpretation_t kInterp = SCHEME == HR_S_FP8E4M3 ? __NV_E4M3 : __NV_E5M2;
#pragma unroll 2
  for (uint32_t e = ctid * 8; e < h.n_el; e += kChunkStride) {
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
    st_v4(h.out + 2ull * e, o[0], o[1], o[2], o[3]);
  }
}

// MXFP8 (R31): E4M3 value (exact, via fp16) times 2^(s - 127) (exact in fp32: >= 2^-136), then one RNE
// to the output dtype; the 8 elements of a chunk share one block (chunks are 8-aligned, blocks 32)
template <int DT>
__device__ __forceinline__ void decode_mxfp8(const TileHdr& h, const uint8_t* codes, const uint8_t* meta, int ctid) {
  const uint8_t* sc = meta + h.meta_off;
#pragma unroll 2
  for (uint32_t e = ctid * 8; e < h.n_el; e += kChunkStride) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    const uint32_t sb = sc[e >> 5];
    const float m = sb ? __uint_as_float(sb << 23) : __uint_as_float(0x00400000u);  // 2^(s-127); s = 0: 2^-127
    const uint32_t w[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)w[i], __NV_E4M3);  // exact
      const float2 f = __fmul2_rn(__half22float2(*reinterpret_cast<__half2*>(&hr)), make_float2(m, m));
      o[i] = pack2<DT>(f.x, f.y);
    }
    st_v4(h.out + 2ull * e, o[0], o[1], o[2], o[3]);
  }
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

template <int DT, int M>
__device__ __forceinline__ void decode_gse(const TileHdr& h, const uint8_t* codes, uint32_t record, int ctid) {
  // byte = s | idx (7-M bits) | f (M bits); value = f * T[byte >> M] with T[(s << e) | idx] =
  // (-1)^s 2^(G_idx - (M-1)), the fp32 table at record + 16 (record: 256-B-aligned shared address).
  // fma(f, T, +0) is that exact product, except that the -0 of a (s=1, f=0) byte becomes +0: field 0
  // decodes to +0.  The table address of byte i is built by one PRMT: low byte = 16 + 4*(byte >> M),
  // upper bytes from `record`.
  constexpr uint32_t fmask = ((1u << M) - 1u) * 0x01010101u;
  constexpr uint32_t omask = ((0xFFu >> M) << 2) * 0x01010101u;
#pragma unroll 2
  for (uint32_t e = ctid * 8; e < h.n_el; e += kChunkStride) {
    const uint2 c = *reinterpret_cast<const uint2*>(codes + e);
    const uint32_t fx = c.x & fmask, fy = c.y & fmask;  // f < 2^M < 128: exact through I2F.S8
    const uint32_t ox = ((c.x >> (M - 2)) & omask) + 0x10101010u, oy = ((c.y >> (M - 2)) & omask) + 0x10101010u;
    float f[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[i] = __fmaf_rn(s8f(fx, i), lds_f32(__byte_perm(ox, record, 0x7650u | i)), 0.f);
      f[4 + i] = __fmaf_rn(s8f(fy, i), lds_f32(__byte_perm(oy, record, 0x7650u | i)), 0.f);
    }
    st_v4(h.out + 2ull * e, pack2<DT>(f[0], f[1]), pack2<DT>(f[2], f[3]), pack2<DT>(f[4], f[5]),
          pack2<DT>(f[6], f[7]));
  }
}

template <int DT>
__device__ __forceinline__ void consume(const AsmParams& p, const Smem& sm, int warp, int lane) {
  const int ctid = warp * 32 + lane;
  uint64_t t0, t1;
  my_tiles(p, t0, t1);
  for (uint64_t i = 0; p.sched || i < t1 - t0; ++i) {
    const int stage = (int)(i % kAsmStages);
    mbar_wait(&sm.full()[stage], (uint32_t)((i / kAsmStages) & 1));
    const TileHdr h = sm.hdr()[stage];
    if (h.n_el == 0) break;  // the producer's end marker (tail-balanced launches)
    const uint8_t* codes = sm.codes(stage);
    const uint8_t* meta = sm.meta(stage);
    switch (h.scheme) {
      case HR_S_PASS16:
        if (warp == 0 && lane == 0) {
          bulk_s2g(h.out, codes, 2 * h.n_el);
          bulk_wait_read_all();  // the stage is released below
        }
        break;
      case HR_S_INT8:
        decode_int8<DT>(h, codes, meta, ctid, p.g_shift);
        break;
      case HR_S_INT4:
        decode_int4<DT>(h, codes, meta, ctid, p.g_shift);
        break;
      case HR_S_FP8E4M3:
        decode_fp8<DT, HR_S_FP8E4M3>(h, codes, ctid);
        break;
      case HR_S_FP8E5M2:
        decode_fp8<DT, HR_S_FP8E5M2>(h, codes, ctid);
        break;
      case HR_S_MXFP8:
        decode_mxfp8<DT>(h, codes, meta, ctid);
        break;
      case HR_S_GSE8:
        if (p.gse_m == 3)
          decode_gse<DT, 3>(h, codes, smem_addr(meta), ctid);
        else if (p.gse_m == 4)
          decode_gse<DT, 4>(h, codes, smem_addr(meta), ctid);
        else
          decode_gse<DT, 5>(h, codes, smem_addr(meta), ctid);
        break;
      default:
        break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty()[stage]);
  }
  if (warp == 0 && lane == 0) bulk_wait_all();
}

template <int DT>
#ifndef HARAG_MIN_BLOCKS
#define HARAG_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kAsmThreads, HARAG_MIN_BLOCKS) assemble_kv_kernel(const __grid_constant__ AsmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem sm{smem_raw, p.meta_stage};
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    if (smem_addr(smem_raw) & 255u) __trap();  // GSE-8 table addressing needs 256-B-aligned meta stages
    for (int s = 0; s < kAsmStages; ++s) {
      mbar_init(&sm.full()[s], 1);
      mbar_init(&sm.empty()[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) produce(p, sm);
  } else {
    consume<DT>(p, sm, warp - 1, lane);
  }
}

int g_num_sms = 0;
constexpr uint32_t kMaxMetaStage = 2 * kAsmCodeStage / 32 * 8 / 2 + 256;  // INT4 at G = 32

int ctas_per_sm(size_t smem) {
  static int cache_bytes[8] = {0}, cache_val[8] = {0};
  for (int i = 0; i < 8; ++i)
    if (cache_bytes[i] == (int)smem) return cache_val[i];
  int n = 0;
  HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, assemble_kv_kernel<HR_BF16>, kAsmThreads, smem));
  for (int i = 0; i < 8; ++i)
    if (cache_bytes[i] == 0) {
      cache_bytes[i] = (int)smem, cache_val[i] = n;
      break;
    }
  return n < 1 ? 1 : n;
}

}  // namespace

int assemble_ctas_per_sm() {
  if (!g_num_sms) {
    const int mx = (int)smem_bytes(kMaxMetaStage);
    HR_CUDA(cudaFuncSetAttribute(assemble_kv_kernel<HR_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HR_CUDA(cudaFuncSetAttribute(assemble_kv_kernel<HR_FP16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    int dev = 0;
    HR_CUDA(cudaGetDevice(&dev));
    HR_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return ctas_per_sm(smem_bytes(256));
}

void launch_assemble(AsmParams p, uint32_t scheme_mask, cudaStream_t st, int grid_ctas) {
  assemble_ctas_per_sm();
  // tile: 16 KB of codes per stage for every mix (8-bit: 16384 elements; PASS16 forces 8192)
  p.tile_e = (scheme_mask & (1u << HR_S_PASS16)) ? (uint32_t)kAsmMaxTileE / 2 : (uint32_t)kAsmMaxTileE;
  p.tiles_per_slab = (p.slab + p.tile_e - 1) / p.tile_e;
  p.n_tiles = (uint64_t)p.n_desc * p.L * p.Hl * p.tiles_per_slab;
  if (p.n_tiles == 0) return;
  // meta window per stage: the tile's groups (+16-B alignment slack) or the GSE-8 record
  uint32_t meta = 0;
  const uint32_t groups = p.tile_e >= p.G ? p.tile_e / p.G : 1;
  if (scheme_mask & (1u << HR_S_INT8)) meta = std::max(meta, 4 * groups + 32);
  if (scheme_mask & (1u << HR_S_INT4)) meta = std::max(meta, 8 * groups + 32);
  if (scheme_mask & (1u << HR_S_GSE8)) meta = std::max(meta, p.meta_stride[HR_S_GSE8]);
  if (scheme_mask & (1u << HR_S_MXFP8)) meta = std::max(meta, p.tile_e / 32 + 32);
  p.meta_stage = (meta + 255) / 256 * 256;  // 256-B-aligned records (GSE-8 table addressing)
  require(p.meta_stage <= kMaxMetaStage, HR_EINVAL, "group too small for the assemble tile");
  const size_t smem = smem_bytes(p.meta_stage);
  uint64_t grid = grid_ctas > 0 ? (uint64_t)grid_ctas : (uint64_t)g_num_sms * ctas_per_sm(smem);
  if (grid > p.n_tiles) grid = p.n_tiles;
  // tail balancing: the last dyn_pct % of the tiles in ~dyn_per_cta chunks per CTA
  if (p.sched && p.dyn_pct && p.n_tiles >= 4 * grid) {
    p.dyn_tiles = p.n_tiles * p.dyn_pct / 100;
    p.dyn_chunk = (uint32_t)std::max<uint64_t>(1, p.dyn_tiles / (grid * std::max(1u, p.dyn_per_cta)));
  } else {
    p.sched = nullptr;
  }
  if (p.dtype == HR_BF16)
    assemble_kv_kernel<HR_BF16><<<(unsigned)grid, kAsmThreads, smem, st>>>(p);
  else
    assemble_kv_kernel<HR_FP16><<<(unsigned)grid, kAsmThreads, smem, st>>>(p);
  HR_CUDA(cudaGetLastError());
}

}  // namespace harag
