// Host cost of cudaLaunchKernel vs kernel-parameter size on this box, with the GPU idle between
// launches (the single-request latency case of hr_assemble_kv: descriptors carried inline in the
// parameters) and with an event record before the launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

template <int N>
struct P {
  unsigned char b[N];
};
template <int N>
__global__ void k(const __grid_constant__ P<N> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[0] == 123) *out = 1;
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int N>
void probe(int* out, cudaStream_t st, cudaEvent_t ev) {
  P<N> p{};
  for (int mode = 0; mode < 2; ++mode) {
    double tot = 0;
    const int reps = 200;
    for (int i = 0; i < reps + 10; ++i) {
      cudaStreamSynchronize(st);
      if (mode) cudaEventRecord(ev, st);
      const double a = now_us();
      k<N><<<148, 928, 0, st>>>(p, out);
      const double b = now_us();
      if (i >= 10) tot += b - a;
    }
    cudaStreamSynchronize(st);
    printf("params %5d B %s: cudaLaunchKernel %.2f us\n", N, mode ? "after event record" : "idle stream       ",
           tot / reps);
  }
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  probe<64>(out, st, ev);
  probe<1024>(out, st, ev);
  probe<2720>(out, st, ev);
  probe<4000>(out, st, ev);
  probe<8000>(out, st, ev);
  probe<16000>(out, st, ev);
  return 0;
}
