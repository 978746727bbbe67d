// Pageable -> pinned bounce -> HBM pipeline of the host-tier streamer, in isolation: the
// store's CopyPool copies each piece of a pageable item into a pinned bounce buffer and a
// cudaMemcpyAsync moves it to the device while the next piece is copied.  Sweeps worker count and
// piece size; prints the achieved link GB/s (bytes / wall time of the whole stream).
//   nvcc -O3 -std=c++17 -Ipaper_2510_20878_b200/csrc -o tools/bounce_bench tools/bounce_bench.cpp -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pool.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t item = 17301504;            // one Llama-3-8B INT8 item blob (16.5 MiB)
  const size_t n_items = argc > 1 ? atoi(argv[1]) : 400;  // distinct pageable items streamed
  const size_t src_bytes = 256 * item;     // 4.4 GB of pageable backing, cycled
  uint8_t* src = (uint8_t*)aligned_alloc(4096, src_bytes);
  memset(src, 7, src_bytes);
  const int slots = 8;
  std::vector<uint8_t*> bounce(slots), dev(slots);
  std::vector<cudaEvent_t> copied(slots);
  for (int s = 0; s < slots; ++s) {
    cudaHostAlloc((void**)&bounce[s], item, cudaHostAllocPortable);
    cudaMalloc(&dev[s], item);
    cudaEventCreateWithFlags(&copied[s], cudaEventDisableTiming);
  }
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  // pinned DMA alone
  double t0 = now();
  for (size_t i = 0; i < n_items; ++i) cudaMemcpyAsync(dev[i % slots], bounce[i % slots], item, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  printf("pinned DMA alone: %.1f GB/s\n", n_items * item / (now() - t0) / 1e9);
  // the driver's own staging of a pageable source (cudaMemcpyAsync straight from pageable memory)
  t0 = now();
  for (size_t i = 0; i < n_items / 4; ++i)
    cudaMemcpyAsync(dev[i % slots], src + (i % 256) * item, item, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  printf("pageable cudaMemcpyAsync (driver staging): %.1f GB/s\n", n_items / 4 * item / (now() - t0) / 1e9);
  {  // host copy alone (no DMA), whole items, all workers
    harag::CopyPool pool(15, 2000, true);
    t0 = now();
    for (size_t i = 0; i < n_items; ++i) pool.copy(bounce[i % slots], src + (i % 256) * item, item);
    printf("host bounce copy alone (16 threads, NT): %.1f GB/s\n", n_items * item / (now() - t0) / 1e9);
  }
  const bool sweep_pieces = getenv("BB_PIECES") != nullptr;
  const int reps = getenv("BB_REPS") ? atoi(getenv("BB_REPS")) : 1;
  for (int rep = 0; rep < reps; ++rep)
  for (unsigned workers : {3u, 5u, 7u, 9u, 11u, 15u}) {
    for (int nt : {0, 1}) {
      harag::CopyPool pool(workers, 2000, nt != 0);
      printf("-- %s copies\n", nt ? "non-temporal" : "memcpy");
      std::vector<size_t> pieces = {item};
      if (sweep_pieces) pieces = {(size_t)4 << 20, (size_t)8 << 20, item};
      for (size_t piece : pieces) {
        std::vector<bool> used(slots, false);
        double t1 = now();
        double host_copy = 0;
        for (size_t i = 0; i < n_items; ++i) {
          const int s = (int)(i % slots);
          if (used[s]) cudaEventSynchronize(copied[s]);
          const uint8_t* sp = src + (i % 256) * item;
          for (size_t off = 0; off < item; off += piece) {
            const size_t n = std::min(piece, item - off);
            double a = now();
            pool.copy(bounce[s] + off, sp + off, n);
            host_copy += now() - a;
            cudaMemcpyAsync(dev[s] + off, bounce[s] + off, n, cudaMemcpyHostToDevice, st);
          }
          cudaEventRecord(copied[s], st);
          used[s] = true;
        }
        cudaStreamSynchronize(st);
        const double dt = now() - t1;
        printf("workers %2u piece %5zu KiB: link %.1f GB/s, host copy %.1f GB/s (%.0f%% of wall)\n", workers,
               piece >> 10, n_items * item / dt / 1e9, n_items * item / host_copy / 1e9, 100 * host_copy / dt);
      }
    }
  }
  return 0;
}
