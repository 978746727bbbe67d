// Achievable HBM bandwidth on this B200 for the traffic mixes of the assemble
// kernel (context for the roofline): copy 1:1, widen 1:2 (read 1 B, write 2 B
// per element, like an 8-bit -> 16-bit decode), write-only, read-only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membw tools/membw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy_k(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void widen_k(const uint2* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint2 v = a[i];
    b[i] = make_uint4(__byte_perm(v.x, 0, 0x4140), __byte_perm(v.x, 0, 0x4342), __byte_perm(v.y, 0, 0x4140),
                      __byte_perm(v.y, 0, 0x4342));
  }
}
__global__ void write_k(uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_uint4(i, i, i, i);
}
__global__ void read_k(const uint4* __restrict__ a, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = a[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const size_t bytes = 8ull << 30;  // 8 GiB buffers (>> L2)
  uint8_t *a, *b;
  uint32_t* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grids[3] = {sms * 4, sms * 8, sms * 16};
  for (int mode = 0; mode < 4; ++mode) {
    double best = 0;
    for (int gi = 0; gi < 3; ++gi) {
      for (int rep = 0; rep < 6; ++rep) {
        double moved = 0;
        cudaEventRecord(e0);
        if (mode == 0) {
          size_t n = bytes / 2 / 16;  // copy 4 GiB -> 4 GiB
          copy_k<<<grids[gi], 256>>>((const uint4*)a, (uint4*)b, n);
          moved = 2.0 * n * 16;
        } else if (mode == 1) {
          size_t n = bytes / 2 / 16;  // read 4 GiB of bytes... n uint2 reads (8 B), n uint4 writes (16 B)
          widen_k<<<grids[gi], 256>>>((const uint2*)a, (uint4*)b, n);
          moved = 24.0 * n;
        } else if (mode == 2) {
          size_t n = bytes / 16;
          write_k<<<grids[gi], 256>>>((uint4*)b, n);
          moved = 16.0 * n;
        } else {
          size_t n = bytes / 16;
          read_k<<<grids[gi], 256>>>((const uint4*)a, n, sink);
          moved = 16.0 * n;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && moved / ms / 1e6 > best) best = moved / ms / 1e6;
      }
    }
    const char* names[4] = {"copy 1:1 (read+write)", "widen 1:2 (read 1 B, write 2 B)", "write only", "read only"};
    printf("{\"pattern\": \"%s\", \"GBps\": %.1f}\n", names[mode], best);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
