// NUMA locality of a rank's host tiers: the CPUs NVML reports as local
// to the store's GPU, and an RAII guard that runs the calling thread on them while the store
// allocates or first touches host memory (pinned tier, pinned / pageable backing, bounce buffers),
// so the kernel's first-touch policy places those pages on the GPU's node.  NVML is loaded at run
// time (dlopen), so the library has no link-time dependency on it; without NVML the list is empty
// and nothing is bound.
#pragma once

#include <sched.h>

#include <vector>

namespace harag {

// CPUs local to CUDA device `device` (NVML nvmlDeviceGetCpuAffinity), restricted to the CPUs this
// process may run on.  Empty when NVML is unavailable or every allowed CPU is local (nothing to bind).
std::vector<int> gpu_local_cpus(int device);

// Binds the calling thread to `cpus` for its lifetime (no-op when cpus is empty).
class CpuBind {
 public:
  explicit CpuBind(const std::vector<int>& cpus);
  ~CpuBind();
  CpuBind(const CpuBind&) = delete;
  CpuBind& operator=(const CpuBind&) = delete;

 private:
  bool active_ = false;
  cpu_set_t saved_;
};

}  // namespace harag
