// Analysis tooling: exponent histograms and
// per-scheme compression error, Eq..
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "harag.h"

namespace harag {

// Encode one item (this rank's heads of src [L][H][T][D]) with `scheme`, decode it with the
// assemble kernel, and return out[0] = sum of squared errors (fp64), out[1] = max |error|.
// Synchronous on `st`.
void scheme_error(const hr_store_config& cfg, uint32_t scheme, const void* src, double out[2], cudaStream_t st);

// hist[b] += number of 16-bit values of src[0..n) whose biased exponent field is b.
void launch_exponent_hist(uint32_t dtype, const void* src, uint64_t n, unsigned long long* hist, cudaStream_t stream);

// Number of fp64 partials launch_error uses for n_elems elements (scratch = 2 * that doubles).
uint32_t error_partials(uint64_t n_elems);

// out[0] = sum of (x - y)^2 in fp64, out[1] = max |x - y|, over this rank's heads [h0, h0+Hl)
// of x ([L][H][slab]) against y ([L][Hl][slab]).
void launch_error(const uint16_t* x, const uint16_t* y, uint32_t L, uint32_t H, uint32_t Hl, uint32_t h0,
                  uint64_t slab, uint32_t dtype, double* partials, uint32_t n_part, double* out, cudaStream_t stream);

// Value-distribution guard statistics of one item (R29): src = [n_slabs][slab] 16-bit values
// (an item's ALL-heads source); stats[0] += values GSE-8 (layout 1+e_bits+m_bits) flushes to zero,
// stats[1] = max(stats[1], fp32 bits of max |x|).  Stream-ordered.
void launch_guard(uint32_t dtype, const void* src, uint64_t n_slabs, uint64_t slab, uint32_t e_bits,
                  uint32_t m_bits, unsigned long long* stats, cudaStream_t st);

}  // namespace harag
