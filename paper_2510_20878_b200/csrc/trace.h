// NVTX ranges of the store runtime (header-only NVTX v3 from the CUDA toolkit: no link dependency;
// the ranges cost a load and a branch unless a profiler such as Nsight Systems / ncu is attached).
// Ranges: hr_build, hr_assemble_kv > {plan, launch_a, host_tier_stream > {bounce, launch_b}},
// hr_replace > {migrate}, hr_attend.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace harag {

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace harag
