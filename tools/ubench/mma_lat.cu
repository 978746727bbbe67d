// Micro-benchmark: completion time of a batch of tcgen05.mma (kind::f16, M = 128, K = 16 each) issued by
// one thread, as a function of N, A source (shared memory / TMEM) and accumulator dependence.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_lat.cu -o mma_lat && ./mma_lat
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(uint32_t n, uint32_t m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss_el(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts_el(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}
template <int N, int CNT, bool TS>
__device__ __forceinline__ void unrolled(uint32_t tm, uint32_t a0, uint32_t b0) {
  constexpr uint32_t id = idesc(N, 128);
#pragma unroll
  for (int s = 0; s < CNT; ++s) {
    const uint64_t bd = desc_sw128(b0 + (s & 3) * 32);
    if (TS) mma_ts_el(tm, tm + 256 + (s & 7) * 8, bd, id, s > 0);
    else mma_ss_el(tm, desc_sw128(a0 + (s & 3) * 32), bd, id, s > 0);
  }
}
// mode: 0 SS same D, 1 TS same D, 2 SS independent D (chains = nchain round-robin), 3 TS independent
__global__ void k(int mode, int n, int count, int nchain, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  long long best = 1ll << 60;
  for (int rep = 0; rep < 5; ++rep) {
    if (mode >= 4 && threadIdx.x < 32) {  // warp-uniform issue, elect.sync per MMA, compile-time unrolled
      const uint32_t a0 = sa(sm), b0 = sa(sm + 32768);
      long long t0 = clock64();
      if (mode == 4) unrolled<64, 8, false>(tm, a0, b0);
      if (mode == 5) unrolled<64, 8, true>(tm, a0, b0);
      if (mode == 6) unrolled<256, 8, false>(tm, a0, b0);
      if (mode == 7) unrolled<144, 4, true>(tm, a0, b0);
      if (mode == 8) unrolled<64, 32, false>(tm, a0, b0);
      if (mode == 9) unrolled<128, 8, true>(tm, a0, b0);
      if (mode == 10) unrolled<128, 32, true>(tm, a0, b0);
      if (mode == 11) unrolled<64, 32, true>(tm, a0, b0);
      if (mode == 12) unrolled<256, 32, true>(tm, a0, b0);
      if (mode == 13) unrolled<16, 32, true>(tm, a0, b0);
      if (mode == 14) unrolled<16, 4, true>(tm, a0, b0);
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n}" ::"r"(sa(&bar)),
                     "r"(rep & 1));
        long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
      }
      __syncwarp();
    } else if (mode < 4 && threadIdx.x == 0) {
      const uint32_t id = idesc(n, 128);
      const uint32_t a0 = sa(sm), b0 = sa(sm + 32768);
      long long t0 = clock64();
      for (int i = 0; i < count; ++i) {
        const int c = (mode >= 2) ? i % nchain : 0, s = (mode >= 2) ? i / nchain : i;
        const uint32_t d = tm + c * n;  // chains: disjoint column ranges (n * nchain <= 256)
        const uint64_t bd = desc_sw128(b0 + (s & 3) * 32);
        if (mode == 0 || mode == 2)
          mma_ss(d, desc_sw128(a0 + (s & 3) * 32), bd, id, s > 0);
        else
          mma_ts(d, tm + 256 + (s & 7) * 8, bd, id, s > 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
      asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(sa(&bar)),
                   "r"(rep & 1));
      long long t1 = clock64();
      if (t1 - t0 < best) best = t1 - t0;
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) *out = best;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  struct C { int mode, n, count, nchain; const char* what; } cs[] = {
      {0, 64, 1, 1, "SS N64 x1"},         {0, 64, 8, 1, "SS N64 x8 dep"},      {1, 64, 8, 1, "TS N64 x8 dep"},
      {0, 128, 8, 1, "SS N128 x8 dep"},   {0, 256, 8, 1, "SS N256 x8 dep"},    {1, 144, 4, 1, "TS N144 x4 dep"},
      {1, 128, 8, 1, "TS N128 x8 dep"},   {1, 256, 8, 1, "TS N256 x8 dep"},
      {2, 64, 8, 2, "SS N64 2 chains x4"}, {2, 64, 16, 2, "SS N64 2 chains x8"}, {2, 64, 16, 4, "SS N64 4 chains x4"},
      {3, 64, 16, 2, "TS N64 2 chains x8"}, {4, 64, 8, 1, "uni SS N64 x8"}, {5, 64, 8, 1, "uni TS N64 x8"},
      {6, 256, 8, 1, "uni SS N256 x8"}, {7, 144, 4, 1, "uni TS N144 x4"}, {8, 64, 32, 1, "uni SS N64 x32"}, {0, 64, 32, 1, "SS N64 x32 dep"},   {0, 256, 32, 1, "SS N256 x32 dep"},
      {9, 128, 8, 1, "uni TS N128 x8"}, {10, 128, 32, 1, "uni TS N128 x32"}, {11, 64, 32, 1, "uni TS N64 x32"},
      {12, 256, 32, 1, "uni TS N256 x32"}, {13, 16, 32, 1, "uni TS N16 x32"}, {14, 16, 4, 1, "uni TS N16 x4"},
  };
  for (auto& c : cs) {
    k<<<1, 128, 65536>>>(c.mode, c.n, c.count, c.nchain, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", c.what, cudaGetErrorString(e)); return 1; }
    printf("%-22s %6lld cycles  (%5.1f per MMA, ideal %5.1f)\n", c.what, *out, (double)*out / c.count, 128.0 * c.n / 256);
  }
  return 0;
}
