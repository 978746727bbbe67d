// Analysis tooling, host side: the compression error of one
// item under one scheme, Eq., computed entirely on the GPU with the
// store's own quantize and assemble kernels (encode -> decode -> error reduce).
#include "analysis.h"

#include <cuda_runtime.h>

#include <vector>

#include "common.h"
#include "kernels.h"
#include "layout.h"

namespace harag {

namespace {
struct DevBuf {  // freed on every exit path
  void* p = nullptr;
  explicit DevBuf(size_t n) { HR_CUDA(cudaMalloc(&p, n ? n : 1)); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
}  // namespace

void scheme_error(const hr_store_config& cfg, uint32_t scheme, const void* src, double out[2], cudaStream_t st) {
  require(scheme < HR_N_SCHEMES, HR_EINVAL, "unknown scheme");
  require(src != nullptr && out != nullptr, HR_EINVAL, "NULL pointer");
  require(reinterpret_cast<uintptr_t>(src) % 16 == 0, HR_EINVAL, "source must be 16-byte aligned");
  const Layout lay = make_layout(cfg);
  HR_CUDA(cudaSetDevice(cfg.device));
  const uint64_t item = lay.item_bytes(scheme);
  const uint64_t dec = 2 * lay.n_slabs() * lay.slab();
  const uint32_t n_part = error_partials(lay.n_slabs() * lay.slab());
  DevBuf blob(item), y(dec), err(sizeof(int)), gse(sizeof(int) * 2 * lay.n_slabs()), desc(sizeof(AsmDesc)),
      part(sizeof(double) * (2 * n_part + 2));
  HR_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), st));
  HR_CUDA(cudaMemsetAsync(blob.p, 0, item, st));
  QuantParams q{};
  q.src = static_cast<const uint16_t*>(src);
  q.dst = blob.as<uint8_t>();
  q.L = lay.L, q.H = lay.H, q.Hl = lay.Hl, q.h0 = lay.h0, q.T = lay.T, q.D = lay.D, q.G = lay.G;
  q.gse_e = lay.gse_e, q.gse_m = lay.gse_m, q.dtype = lay.dtype, q.scheme = scheme;
  q.g_shift = (uint32_t)__builtin_ctz(lay.G);
  q.code_bytes_slab = lay.code_bytes_slab(scheme);
  q.meta_offset = lay.meta_offset(scheme);
  q.meta_stride = lay.meta_stride(scheme);
  q.err = err.as<int>();
  q.gse_range = gse.as<int>();
  launch_quantize(&q, 1, st);
  AsmDesc d{};
  d.codes = blob.as<uint8_t>();
  d.meta = blob.as<uint8_t>() + lay.meta_offset(scheme);
  d.out = y.as<uint8_t>();
  d.count = nullptr;
  d.slot = 0;
  d.scheme = scheme;
  HR_CUDA(cudaMemcpyAsync(desc.p, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  AsmParams p{};
  p.descs = desc.as<AsmDesc>();
  p.n_desc = 1;
  p.L = lay.L, p.Hl = lay.Hl, p.T = lay.T, p.D = lay.D, p.k = 1, p.G = lay.G;
  p.g_shift = (uint32_t)__builtin_ctz(lay.G);
  p.gse_m = lay.gse_m;
  p.dtype = lay.dtype;
  p.slab = (uint32_t)lay.slab();
  for (uint32_t s = 0; s < HR_N_SCHEMES; ++s) p.meta_stride[s] = (uint32_t)lay.meta_stride(s);
  launch_assemble(p, 1u << scheme, st);
  double* res = part.as<double>() + 2 * n_part;
  launch_error(static_cast<const uint16_t*>(src), y.as<uint16_t>(), lay.L, lay.H, lay.Hl, lay.h0, lay.slab(),
               lay.dtype, part.as<double>(), n_part, res, st);
  HR_CUDA(cudaGetLastError());
  int e = 0;
  HR_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  HR_CUDA(cudaMemcpyAsync(out, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  HR_CUDA(cudaStreamSynchronize(st));
  require(e == 0, HR_EINVAL, "NaN/Inf in the source item (rejected at ingestion, S:30)");
}

}  // namespace harag
