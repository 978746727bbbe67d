// Host copy micro-benchmark for the pageable -> pinned bounce of the host-tier streamer
// (P:213).  Measures memcpy vs non-temporal (streaming-store) copies from a large pageable
// buffer into a pinned-sized destination with 1..N threads, and the H2D DMA running at the
// same time (the real contention: DMA reads host DRAM while the CPU copies).
//   nvcc -O3 -o tools/hostcopy tools/hostcopy.cpp -lpthread && tools/hostcopy
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target("avx2"))) static void copy_nt(void* dst, const void* src, size_t n) {
  auto* d = (__m256i*)dst;
  auto* s = (const __m256i*)src;
  size_t v = n / 32;
  for (size_t i = 0; i < v; i += 4) {
    __m256i a = _mm256_loadu_si256(s + i), b = _mm256_loadu_si256(s + i + 1);
    __m256i c = _mm256_loadu_si256(s + i + 2), e = _mm256_loadu_si256(s + i + 3);
    _mm256_stream_si256(d + i, a);
    _mm256_stream_si256(d + i + 1, b);
    _mm256_stream_si256(d + i + 2, c);
    _mm256_stream_si256(d + i + 3, e);
  }
  _mm_sfence();
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t total = (argc > 1 ? atoll(argv[1]) : 16ull) << 30;  // pageable source GiB
  const size_t piece = 4u << 20;
  uint8_t* src = (uint8_t*)aligned_alloc(4096, total);
  for (size_t i = 0; i < total; i += 4096) src[i] = (uint8_t)i;  // touch
  memset(src, 1, total);
  const size_t ring = 64u << 20;
  uint8_t* pin = nullptr;
  cudaHostAlloc((void**)&pin, ring, cudaHostAllocPortable);
  uint8_t* dev = nullptr;
  cudaMalloc(&dev, ring);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  unsigned hw = std::thread::hardware_concurrency();
  printf("hw threads %u, source %zu GiB pageable, pieces %zu MiB\n", hw, total >> 30, piece >> 20);
  for (int mode = 0; mode < 2; ++mode) {
    for (unsigned t : {1u, 2u, 4u, 8u, 12u, 15u}) {
      if (t > hw) continue;
      for (int dma = 0; dma < 2; ++dma) {
        size_t off = 0;
        double t0 = now();
        size_t moved = 0;
        while (off + piece * t <= total && moved < (8ull << 30)) {
          std::vector<std::thread> th;
          for (unsigned i = 0; i < t; ++i)
            th.emplace_back([&, i] {
              uint8_t* d = pin + ((off / piece + i) % (ring / piece)) * piece;
              if (mode) copy_nt(d, src + off + i * piece, piece);
              else memcpy(d, src + off + i * piece, piece);
            });
          for (auto& x : th) x.join();
          if (dma) cudaMemcpyAsync(dev, pin + ((off / piece) % (ring / piece)) * piece, piece * t,
                                   cudaMemcpyHostToDevice, st);
          off += piece * t;
          moved += piece * t;
          if (dma && (off / piece) % 8 == 0) cudaStreamSynchronize(st);
        }
        cudaStreamSynchronize(st);
        double dt = now() - t0;
        printf("%-8s threads %2u dma %d: %6.1f GB/s\n", mode ? "stream" : "memcpy", t, dma, moved / dt / 1e9);
      }
    }
  }
  // DMA alone
  double t0 = now();
  for (int i = 0; i < 64; ++i) cudaMemcpyAsync(dev, pin, ring, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  printf("pinned H2D alone: %.1f GB/s\n", 64.0 * ring / (now() - t0) / 1e9);
  return 0;
}
