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

constexpr int kAsmThreads = 288;       // 1 producer warp + 8 consumer warps
constexpr int kAsmTileE = 8192;       // elements per tile (16 KB of 16-bit output)
constexpr int kAsmStages = 4;         // shared-memory ring depth
constexpr int kAsmCodeStage = 2 * kAsmTileE;           // PASS16 worst case
constexpr int kAsmMetaStage = 2048 + 64;               // INT4 at G=32 worst case + 16-B window slack

struct AsmParams {
  const AsmDesc* descs;
  uint32_t n_desc;
  uint32_t L, Hl, T, D, k, G;
  uint32_t g_shift;          // log2(G) (G is a power of two)
  uint32_t gse_m;
  uint32_t dtype;            // hr_dtype of the output
  uint32_t slab;             // T*D
  uint32_t tiles_per_slab;   // ceil(slab / kAsmTileE)
  uint64_t n_tiles;          // n_desc * L * Hl * tiles_per_slab
  uint32_t meta_stride[6];   // per scheme, bytes per slab record
};

// Launch the fused gather -> unpack -> dequantise -> scatter (+ hotness count).
// grid_ctas <= 0: persistent grid of SMs x resident CTAs.
void launch_assemble(const AsmParams& p, cudaStream_t stream, int grid_ctas = 0);
int assemble_ctas_per_sm();

struct QuantParams {
  const uint16_t* src;       // [L][H][T][D] all heads, source dtype
  uint8_t* dst;              // item blob base
  uint32_t L, H, Hl, h0, T, D, G, gse_e, gse_m, dtype, scheme;
  uint64_t code_bytes_slab, meta_offset, meta_stride;
  int* err;                  // set to 1 on NaN/Inf
};

// a3 + a4: one CTA per (layer, local head) slab.
void launch_quantize(const QuantParams& p, cudaStream_t stream);

}  // namespace harag
