#include "numa.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <pthread.h>

#include <mutex>

namespace harag {

namespace {
using nvmlInit_t = int (*)();
using nvmlByBusId_t = int (*)(const char*, void**);
using nvmlCpuAffinity_t = int (*)(void*, unsigned int, unsigned long*);

struct Nvml {
  nvmlByBusId_t by_bus = nullptr;
  nvmlCpuAffinity_t affinity = nullptr;
  bool ok = false;
};

const Nvml& nvml() {
  static Nvml n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto init = (nvmlInit_t)dlsym(h, "nvmlInit_v2");
    n.by_bus = (nvmlByBusId_t)dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2");
    n.affinity = (nvmlCpuAffinity_t)dlsym(h, "nvmlDeviceGetCpuAffinity");
    n.ok = init && n.by_bus && n.affinity && init() == 0;
  });
  return n;
}
}  // namespace

std::vector<int> gpu_local_cpus(int device) {
  std::vector<int> out;
  const Nvml& n = nvml();
  if (!n.ok) return out;
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return out;
  }
  void* dev = nullptr;
  if (n.by_bus(bus, &dev) != 0) return out;
  constexpr unsigned kWords = 1024 / (8 * sizeof(unsigned long));
  unsigned long mask[kWords] = {0};
  if (n.affinity(dev, kWords, mask) != 0) return out;
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof allowed, &allowed) != 0) return out;
  int n_allowed = 0;
  for (int c = 0; c < CPU_SETSIZE; ++c) {
    if (!CPU_ISSET(c, &allowed)) continue;
    ++n_allowed;
    if (c < 1024 && (mask[c / (8 * sizeof(unsigned long))] >> (c % (8 * sizeof(unsigned long))) & 1ul))
      out.push_back(c);
  }
  if ((int)out.size() == n_allowed) out.clear();  // every allowed CPU is local: nothing to bind
  return out;
}

CpuBind::CpuBind(const std::vector<int>& cpus) {
  if (cpus.empty()) return;
  if (pthread_getaffinity_np(pthread_self(), sizeof saved_, &saved_) != 0) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus) CPU_SET(c, &set);
  active_ = pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0;
}

CpuBind::~CpuBind() {
  if (active_) pthread_setaffinity_np(pthread_self(), sizeof saved_, &saved_);
}

}  // namespace harag
