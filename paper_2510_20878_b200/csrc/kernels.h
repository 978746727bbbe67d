// Device-side interfaces of the sm_100a kernels (quantize.cu, assemble.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace harag {

// One (request, slot, kind) of an assemble launch: where the item's packed
// blob lives (HBM arena or staging-ring slot) and where its slabs go.
struct AsmDesc {
  const uint8_t* codes;      // codes section of the item blob (this rank's heads)
  const uint8_t* meta;       // meta section
  uint8_t* out;              // K_out[r] or V_out[r]: [L][Hl][k*T][D] of 16-bit
  unsigned long long* count; // hotness delta counter of the item, or nullptr (a1)
  uint32_t slot;             // j: position of the doc in the request
  uint32_t scheme;           // hr_scheme
};

#ifndef HARAG_CONSUMER_WARPS
#define HARAG_CONSUMER_WARPS 28
#endif
constexpr int kAsmThreads = 32 * (1 + HARAG_CONSUMER_WARPS);  // 1 producer warp + consumer warps
#ifndef HARAG_STAGES
#define HARAG_STAGES 4
#endif
#ifndef HARAG_CODE_STAGE
#define HARAG_CODE_STAGE 16384
#endif
constexpr int kAsmStages = HARAG_STAGES;         // shared-memory ring depth
constexpr int kAsmCodeStage = HARAG_CODE_STAGE;  // bytes of packed codes per stage (every scheme mix)
constexpr int kAsmMaxTileE = kAsmCodeStage;      // elements per tile (half when a launch holds PASS16 items)

#ifndef HARAG_ASM_INLINE
#define HARAG_ASM_INLINE 64
#endif
constexpr int kAsmInline = HARAG_ASM_INLINE;  // launches of <= kAsmInline descriptors carry them in the kernel parameters

struct AsmParams {
  const AsmDesc* descs;      // device array, or nullptr: the descriptors are inl[0..n_desc)
  uint32_t n_desc;
  uint32_t L, Hl, T, D, k, G;
  uint32_t g_shift;          // log2(G) (G is a power of two)
  uint32_t gse_m;
  uint32_t dtype;            // hr_dtype of the output
  uint32_t slab;             // T*D
  uint32_t tile_e;           // elements per tile (power of two)
  uint32_t tiles_per_slab;   // ceil(slab / tile_e)
  uint32_t meta_stage;       // bytes of meta window per stage (multiple of 128)
  uint64_t n_tiles;          // n_desc * L * Hl * tiles_per_slab
  uint32_t meta_stride[HR_N_SCHEMES];  // per scheme, bytes per slab record
  // Tail balancing: tiles [n_tiles - dyn_tiles, n_tiles) are claimed in chunks of dyn_chunk through an
  // atomic counter (sched[0]; sched[1] counts producers done, the last one zeroes both), the rest are
  // split in blocks.  sched == nullptr: blocked split only.
  uint32_t* sched;           // [4]: u64 claim counter, u32 done count (zero between launches), or nullptr
  uint32_t dyn_pct;          // input: percent of the tiles claimed dynamically (0: blocked split only)
  uint32_t dyn_per_cta;      // input: dynamic chunks per CTA (sets the chunk size)
  uint64_t dyn_tiles;        // filled in by launch_assemble
  uint32_t dyn_chunk;
  AsmDesc inl[kAsmInline > 0 ? kAsmInline : 1];   // small launches (a single request, a streamed item): no descriptor H2D copy
};

// Launch the fused gather -> unpack -> dequantise -> scatter (+ hotness count).
// scheme_mask: bit s set when some descriptor has scheme s (chooses tile and meta window).
// tile_e, tiles_per_slab, n_tiles and meta_stage are filled in here.
// grid_ctas <= 0: persistent grid of SMs x resident CTAs.
void launch_assemble(AsmParams p, uint32_t scheme_mask, cudaStream_t stream, int grid_ctas = 0);
int assemble_ctas_per_sm();

struct QuantParams {
  const uint16_t* src;       // [L][H][T][D] all heads, source dtype
  uint8_t* dst;              // item blob base
  uint32_t L, H, Hl, h0, T, D, G, gse_e, gse_m, dtype, scheme;
  uint32_t g_shift;          // log2(G)
  uint64_t code_bytes_slab, meta_offset, meta_stride;
  int* err;                  // set to 1 on NaN/Inf
  int* gse_range;            // GSE-8: device scratch int[2 * L * Hl] of THIS item (per-slab exponent range)
};

// a3 + a4 for a batch of items sharing one layout (any scheme mix): one TMA-staged launch per
// batch of up to 32 items (+ a read-only GSE-8 range pass when the batch holds GSE-8 items).
// Padding bytes of the blobs are not written (the caller zero-fills them).
void launch_quantize(const QuantParams* items, int n, cudaStream_t stream);

// Consumer: attention of each request's query rows over its retrieved
// chunks, decoding the packed codes inside the kernel (kernels/attend.cu).
struct AttnParams {
  const AsmDesc* descs;      // [n_req][k][2] (K, V) of HBM-resident items; count = hotness counter or nullptr
  const uint16_t* q;         // [n_req][L][Hl*g][n_q][D]
  uint16_t* o;               // same layout as q
  float* lse;                // [n_req][L][Hl*g][n_q] natural-log sum of exp of the scaled scores, or nullptr
  uint16_t* kv_dump;         // test hook: decoded KV [n_req][2][L][Hl][k*T][D], or nullptr
  uint32_t n_req, k, L, Hl, T, D, g, n_q, M;  // M = g * n_q <= 128; L = layers of this call (window)
  uint32_t l0;               // first store layer of the window (q / o / lse / kv_dump index layers 0..L-1)
  uint32_t G, g_shift, gse_e, gse_m, dtype;
  float scale_log2;          // softmax scale * log2(e)
  uint64_t code_slab[HR_N_SCHEMES];    // per scheme, code bytes per slab
  uint32_t meta_stride[HR_N_SCHEMES];  // per scheme, bytes per slab meta record
  // Key splits (flash-decoding): CTA (unit, s) attends over tiles [s n / n_split, (s+1) n / n_split) of the
  // unit's n key tiles, writes its normalised fp32 partial O and LSE to part_o / part_lse, and the last
  // split to finish (part_cnt[unit], zero between launches) merges the n_split partials into o / lse.
  // prefill form (R30): the question's own K / V [n_req][L][Hl][n_own][D] (16-bit), attended causally after
  // the chunk keys (row t = question token t % n_q sees own keys 0..t % n_q); n_own = 0: chunk keys only
  const uint16_t* own_k;
  const uint16_t* own_v;
  uint32_t n_own;
  uint32_t n_split;          // 1: no split (part_* unused)
  float* part_o;             // [units][n_split][128][D]
  float* part_lse;           // [units][n_split][128]
  uint32_t* part_cnt;        // [units], zero on entry; left zero
};
// splits per unit for a launch of `units` units of `n_tiles` key tiles each on `sms` SMs (1 when the
// units alone fill the machine)
uint32_t attend_splits(uint64_t units, uint32_t n_tiles, int sms);
void launch_attend(const AttnParams& p, cudaStream_t stream);

}  // namespace harag
