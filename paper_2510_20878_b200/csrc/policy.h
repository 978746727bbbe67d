// Host policy of the HA-RAG hot path: Alg. 1 ranking / scheme assignment
// (P:182-206), Alg. 2 lists and its demand-mode state machine
// (P:240-272), hotness counting (a1) and epochs (a9).  Pure host C++, no CUDA.
#pragma once

#include <cstdint>
#include <list>
#include <unordered_map>
#include <vector>

namespace harag {

// Alg. 1 line 1: item ids by (h desc, id asc) (R12).
std::vector<uint32_t> rank_items(const uint64_t* h, uint32_t n);

// Alg. 1 lines 2-8: group boundaries [0, idx_1, ..., n]; idx_j =
// idx_{j-1} + floor(tau_j * n) (R11); the last group takes the remainder.
std::vector<uint64_t> partition_bounds(uint32_t n, const double* tau, uint32_t n_tau);

// Alg. 1: scheme per item id.
std::vector<uint32_t> assign_schemes(const uint64_t* h, uint32_t n, const uint32_t* ladder, uint32_t n_ladder,
                                     const double* tau);

// Value-distribution guard (R29): stats[2i] = values of item i GSE-8
// would flush, stats[2i+1] = fp32 bits of its max |x|.  While an item's scheme would lose values (GSE-8
// flushes some, FP8 E4M3 / E5M2 would saturate: |x| > 448 / 57344) and is not the ladder's first, it
// takes the previous (hotter) ladder scheme.  Every scheme must be one of the ladder's.
std::vector<uint32_t> guard_schemes(const uint32_t* schemes, const uint64_t* stats, uint32_t n, const uint32_t* ladder,
                                    uint32_t n_ladder);

// Alg. 2 step 1 by bytes (R15): longest rank-prefix fitting each budget.
// Returns tier per item: 0 HBM (GPU_LIST), 1 PIN (PIN_LIST), 2 PAGE (PAGE_LIST), 3 DISK (the rest,
// only when page_budget is finite).
std::vector<uint32_t> lists_by_bytes(const std::vector<uint32_t>& order, const uint64_t* sizes,
                                     uint64_t hbm_budget, uint64_t pin_budget, uint64_t page_budget = ~0ull);

// Alg. 2 step 1 by fractions (R13 pairs by name, R14 exclusive end).
// Returns list per item: 0 GPU, 1 PIN, 2 PAGE, 3 DISK.
std::vector<uint32_t> lists_by_fraction(const std::vector<uint32_t>& order, double tau_gpu, double tau_pin,
                                        double tau_page);

// a1 on the host: requests q = base + r with q % world == rank add 1 to both
// items of each doc.
void count_requests(const uint32_t* ids, uint32_t n_req, uint32_t k, uint32_t n_docs, uint64_t req_base,
                    uint32_t rank, uint32_t world, int64_t* delta);

// a9 (R20): h <- (h >> shift) + delta.
void epoch_update(uint64_t* h, const int64_t* delta, uint32_t n, uint32_t shift);

// Alg. 2 step 2 state machine with byte (or count) capacities, inclusive
// promotion and LRU in every queue (R16).
class Alg2 {
 public:
  enum { GPU = 0, PIN = 1, PAGE = 2, DISK = 3 };
  Alg2(uint32_t n_items, const uint32_t* list_of_item, const uint64_t* sizes, uint64_t cap_gpu, uint64_t cap_pin,
       uint64_t cap_page);
  struct Outcome {
    uint32_t hit;
    uint32_t put_mask;
    std::vector<std::pair<uint32_t, uint32_t>> evicted;  // (tier, item)
  };
  Outcome access(uint32_t item);
  void set_lists(const uint32_t* list_of_item);
  std::vector<uint32_t> resident(uint32_t tier) const;  // least -> most recent
  bool contains(uint32_t tier, uint32_t item) const { return q_[tier].pos.count(item) != 0; }

 private:
  struct Queue {
    uint64_t cap = 0, used = 0;
    std::list<uint32_t> lru;  // front = least recent
    std::unordered_map<uint32_t, std::list<uint32_t>::iterator> pos;
  };
  void touch(Queue& q, uint32_t item);
  void put(uint32_t tier, uint32_t item, Outcome& o);
  uint64_t size(uint32_t item) const { return sizes_.empty() ? 1 : sizes_[item]; }
  std::vector<uint32_t> list_;
  std::vector<uint64_t> sizes_;
  Queue q_[3];
};

}  // namespace harag
