// ThreadSanitizer harness of the host-tier streamer's worker pool (paper_2510_20878_b200/csrc/pool.h):
// many back-to-back parallel copies and parallel_for jobs of varying widths, results checked byte
// for byte.  Built and run by tests/test_host_tsan.py with -fsanitize=thread.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pool.h"

int main() {
  harag::CopyPool pool(7);
  std::vector<unsigned char> src(6u << 20), dst(6u << 20);
  for (size_t i = 0; i < src.size(); ++i) src[i] = (unsigned char)(i * 131 + 7);
  int bad = 0;
  for (int it = 0; it < 200; ++it) {
    const size_t n = (size_t)(1u << 20) + (size_t)it * 20011 % (5u << 20);
    std::memset(dst.data(), 0, dst.size());
    pool.copy(dst.data(), src.data(), n);
    bad += std::memcmp(dst.data(), src.data(), n) != 0;
    std::vector<int> hit(pool.size(), 0);
    const unsigned parts = 1 + it % pool.size();
    pool.parallel_for(parts, [&](unsigned p) { hit[p] += 1; });
    for (unsigned p = 0; p < pool.size(); ++p) bad += hit[p] != (p < parts ? 1 : 0);
  }
  std::printf("pool_tsan: %d mismatches\n", bad);
  return bad != 0;
}
