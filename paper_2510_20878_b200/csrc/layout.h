// Packed item blob layout and shape rules, host side.
#pragma once

#include <cstdint>

#include "common.h"

namespace harag {

struct Layout {
  uint32_t L = 0, H = 0, Hl = 0, h0 = 0, D = 0, T = 0, G = 0, gse_e = 4, gse_m = 3, dtype = HR_BF16;

  uint64_t slab() const { return (uint64_t)T * D; }
  uint64_t n_slabs() const { return (uint64_t)L * Hl; }
  // bytes of one slab's codes: PASS16 2 B, INT4 1/2 B, 8-bit 1 B per element
  uint64_t code_bytes_slab(uint32_t s) const {
    return s == HR_S_PASS16 ? 2 * slab() : s == HR_S_INT4 ? slab() / 2 : slab();
  }
  uint64_t meta_raw_slab(uint32_t s) const {
    const uint64_t ng = slab() / G;
    // GSE8: int8 array [2^e] padded to 16 B + fp32 decode table [2^(e+1)]
    return s == HR_S_INT8 ? 4 * ng : s == HR_S_INT4 ? 8 * ng : s == HR_S_GSE8 ? 16 + 4 * (2ull << gse_e)
           : s == HR_S_MXFP8 ? slab() / 32 : 0;
  }
  uint64_t meta_stride(uint32_t s) const { return align_up(meta_raw_slab(s), 16); }
  uint64_t meta_offset(uint32_t s) const { return align_up(n_slabs() * code_bytes_slab(s), 256); }
  uint64_t item_bytes(uint32_t s) const { return align_up(meta_offset(s) + n_slabs() * meta_stride(s), 256); }
  uint64_t kv_bytes(uint32_t k) const { return 2ull * n_slabs() * k * slab(); }  // one of K/V, 16-bit out
};

inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

inline Layout make_layout(const hr_store_config& c) {
  require(c.L > 0 && c.H > 0 && c.D > 0 && c.T > 0, HR_EINVAL, "L, H, D, T must be > 0");
  require(c.world >= 1 && c.rank >= 0 && c.rank < c.world, HR_EINVAL, "bad rank/world");
  require(c.H % (uint32_t)c.world == 0, HR_EINVAL, "H must be divisible by world (KV-head sharding)");
  require(c.D % 8 == 0, HR_EINVAL, "D must be a multiple of 8 (16-byte output rows)");
  require(((uint64_t)c.T * c.D) % 256 == 0, HR_EINVAL, "T*D must be a multiple of 256");
  require(c.dtype == HR_BF16 || c.dtype == HR_FP16, HR_EINVAL, "dtype must be HR_BF16 or HR_FP16");
  Layout l;
  l.L = c.L, l.H = c.H, l.D = c.D, l.T = c.T, l.dtype = c.dtype;
  l.Hl = c.H / c.world;
  l.h0 = (uint32_t)c.rank * l.Hl;
  l.G = c.group ? c.group : c.D;
  require(is_pow2(l.G) && l.G >= 32 && l.slab() % l.G == 0, HR_EINVAL,
          "group must be a power of two >= 32 dividing T*D");
  l.gse_e = c.gse_ebits, l.gse_m = c.gse_mbits;
  // P:327 layouts 1+2+5, 1+3+4, 1+4+3: at most 16 shared exponents per slab
  require(l.gse_e >= 2 && l.gse_e <= 4 && l.gse_e + l.gse_m == 7, HR_EINVAL,
          "GSE layout must be 1+2+5, 1+3+4 or 1+4+3 (P:327)");
  return l;
}

}  // namespace harag
