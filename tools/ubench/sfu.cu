// Micro-benchmark: issue cost of MUFU.EX2, F2FP (bf16x2 pack), FFMA2 and HMNMX2 for W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 sfu.cu -o sfu && ./sfu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  uint32_t h[8] = {0};
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) {
        __nv_bfloat162 p = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]);
        h[i] ^= *reinterpret_cast<uint32_t*>(&p);
        a[i] += 1.0f;
      }
      if (OP == 2) {
        float2 x = __ffma2_rn(make_float2(a[i], a[(i + 1) & 7]), make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
        a[i] = x.x; a[(i + 1) & 7] += x.y;
      }
      if (OP == 3) a[i] = a[i] * 1.0001f + 0.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMallocManaged(&cyc, 8);
  const char* names[] = {"ex2", "f2fp(+fadd)", "ffma2(+fadd)", "ffma"};
  for (int op = 0; op < 4; ++op)
    for (int w : {4, 8, 16, 32}) {
      int iters = 2000;
      void (*kk)(float*, int, long long*) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
      kk<<<148, 32 * w>>>(out, iters, cyc); cudaDeviceSynchronize();
      kk<<<148, 32 * w>>>(out, iters, cyc); cudaDeviceSynchronize();
      double per_warp_instr = (double)*cyc / (iters * 8.0);
      printf("%-14s warps/SM %2d: %6.2f cycles per (8-op group / 8) per warp -> SM issue of this op: %.2f warp-instr/clk\n",
             names[op], w, per_warp_instr, w / per_warp_instr);
    }
  return 0;
}
