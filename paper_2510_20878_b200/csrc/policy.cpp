// Host policy: Alg. 1, Alg. 2, a1 counting, a9 epochs.
#include "policy.h"

#include <algorithm>
#include <cmath>
#include <numeric>

#include "common.h"

namespace harag {

std::vector<uint32_t> rank_items(const uint64_t* h, uint32_t n) {
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  // P:188 "Sort(KVChunks, AF, descending)"; ties by ascending id (R12).
  std::stable_sort(order.begin(), order.end(), [h](uint32_t a, uint32_t b) { return h[a] > h[b]; });
  return order;
}

std::vector<uint64_t> partition_bounds(uint32_t n, const double* tau, uint32_t n_tau) {
  std::vector<uint64_t> b{0};
  for (uint32_t j = 0; j < n_tau; ++j) {
    require(tau[j] >= 0.0 && tau[j] <= 1.0, HR_EINVAL, "tau out of [0,1]");
    // P:190 idx_1 <- tau_1 x 2n; floor (R11), fp64 like the oracle.
    b.push_back(b.back() + (uint64_t)std::floor(tau[j] * (double)n));
  }
  require(b.back() <= n, HR_EINVAL, "taus sum above 1");
  b.push_back(n);
  return b;
}

std::vector<uint32_t> assign_schemes(const uint64_t* h, uint32_t n, const uint32_t* ladder, uint32_t n_ladder,
                                     const double* tau) {
  require(n_ladder >= 1 && n_ladder <= 6, HR_EINVAL, "ladder needs 1..6 schemes");
  std::vector<uint32_t> order = rank_items(h, n);
  std::vector<uint64_t> b = partition_bounds(n, tau, n_ladder - 1);
  std::vector<uint32_t> scheme(n);
  for (uint32_t j = 0; j < n_ladder; ++j)  // P:202-205 Compression(S_j, chunks_j)
    for (uint64_t p = b[j]; p < b[j + 1]; ++p) scheme[order[p]] = ladder[j];
  return scheme;
}

std::vector<uint32_t> lists_by_bytes(const std::vector<uint32_t>& order, const uint64_t* sizes, uint64_t hbm_budget,
                                     uint64_t pin_budget, uint64_t page_budget) {
  std::vector<uint32_t> tier(order.size(), page_budget == ~0ull ? 2u : 3u);
  size_t i = 0;
  const uint64_t budget[3] = {hbm_budget, pin_budget, page_budget};
  for (uint32_t t = 0; t < 3; ++t) {  // longest rank-prefix that fits each budget, no skipping (R15)
    uint64_t used = 0;
    while (i < order.size() && (budget[t] == ~0ull || used + sizes[order[i]] <= budget[t]))
      used += sizes[order[i]], tier[order[i++]] = t;
  }
  return tier;
}

std::vector<uint32_t> lists_by_fraction(const std::vector<uint32_t>& order, double tau_gpu, double tau_pin,
                                        double tau_page) {
  const double t[3] = {tau_gpu, tau_pin, tau_page};
  std::vector<uint64_t> b = partition_bounds((uint32_t)order.size(), t, 3);
  std::vector<uint32_t> list(order.size(), 3);
  for (uint32_t j = 0; j < 3; ++j)
    for (uint64_t p = b[j]; p < b[j + 1]; ++p) list[order[p]] = j;
  return list;
}

void count_requests(const uint32_t* ids, uint32_t n_req, uint32_t k, uint32_t n_docs, uint64_t req_base,
                    uint32_t rank, uint32_t world, int64_t* delta) {
  require(world >= 1 && rank < world, HR_EINVAL, "bad rank/world");
  for (uint32_t r = 0; r < n_req; ++r) {
    if ((req_base + r) % world != rank) continue;
    for (uint32_t j = 0; j < k; ++j) {
      uint32_t d = ids[(uint64_t)r * k + j];
      require(d < n_docs, HR_ENOTFOUND, "doc id out of range");
      delta[2ull * d] += 1;
      delta[2ull * d + 1] += 1;
    }
  }
}

void epoch_update(uint64_t* h, const int64_t* delta, uint32_t n, uint32_t shift) {
  for (uint32_t i = 0; i < n; ++i) {
    int64_t v = (int64_t)(shift >= 64 ? 0 : (h[i] >> shift)) + delta[i];
    require(v >= 0, HR_EINVAL, "negative hotness after epoch");
    h[i] = (uint64_t)v;
  }
}

// ------------------------------------------------------------------- Alg. 2
Alg2::Alg2(uint32_t n_items, const uint32_t* list_of_item, const uint64_t* sizes, uint64_t cap_gpu, uint64_t cap_pin,
           uint64_t cap_page)
    : list_(list_of_item, list_of_item + n_items) {
  if (sizes) sizes_.assign(sizes, sizes + n_items);
  q_[0].cap = cap_gpu;
  q_[1].cap = cap_pin;
  q_[2].cap = cap_page;
  for (uint32_t l : list_) require(l <= 3, HR_EINVAL, "list id must be 0..3");
}

void Alg2::set_lists(const uint32_t* list_of_item) {
  for (size_t i = 0; i < list_.size(); ++i) {
    require(list_of_item[i] <= 3, HR_EINVAL, "list id must be 0..3");
    list_[i] = list_of_item[i];
  }
}

void Alg2::touch(Queue& q, uint32_t item) {  // queue.get(C_i): most recent
  q.lru.splice(q.lru.end(), q.lru, q.pos[item]);
}

void Alg2::put(uint32_t tier, uint32_t item, Outcome& o) {  // "put C_i in queue with LRU"
  Queue& q = q_[tier];
  o.put_mask |= 1u << tier;
  if (q.pos.count(item)) {
    touch(q, item);
    return;
  }
  uint64_t sz = size(item);
  if (sz > q.cap) return;  // can never fit: not cached
  while (q.used + sz > q.cap) {
    uint32_t victim = q.lru.front();
    q.lru.pop_front();
    q.pos.erase(victim);
    q.used -= size(victim);
    o.evicted.emplace_back(tier, victim);
  }
  q.lru.push_back(item);
  q.pos[item] = std::prev(q.lru.end());
  q.used += sz;
}

Alg2::Outcome Alg2::access(uint32_t item) {
  require(item < list_.size(), HR_ENOTFOUND, "item id out of range");
  Outcome o{DISK, 0, {}};
  const uint32_t l = list_[item];
  if (q_[GPU].pos.count(item)) {
    touch(q_[GPU], item);
    o.hit = GPU;
  } else if (q_[PIN].pos.count(item)) {
    touch(q_[PIN], item);
    o.hit = PIN;
    if (l == GPU) put(GPU, item, o);
  } else if (q_[PAGE].pos.count(item)) {
    touch(q_[PAGE], item);
    o.hit = PAGE;
    if (l == GPU) put(GPU, item, o);
    if (l == PIN) put(PIN, item, o);
  } else {  // P:260-270 load from disk, place by list
    o.hit = DISK;
    if (l == GPU) put(GPU, item, o);
    if (l == PIN) put(PIN, item, o);
    if (l == PAGE) put(PAGE, item, o);
  }
  return o;
}

std::vector<uint32_t> Alg2::resident(uint32_t tier) const {
  require(tier < 3, HR_EINVAL, "tier must be 0..2");
  return std::vector<uint32_t>(q_[tier].lru.begin(), q_[tier].lru.end());
}

std::vector<uint32_t> guard_schemes(const uint32_t* schemes, const uint64_t* stats, uint32_t n, const uint32_t* ladder,
                                    uint32_t n_ladder) {
  require(n_ladder >= 1 && n_ladder <= 6, HR_EINVAL, "ladder must hold 1..6 schemes");
  auto unsafe = [](uint32_t s, uint64_t flushed, uint32_t amax_bits) {
    if (s == HR_S_GSE8) return flushed > 0;
    if (s == HR_S_FP8E4M3) return amax_bits > 0x43E00000u;  // |x| > 448
    if (s == HR_S_FP8E5M2) return amax_bits > 0x47600000u;  // |x| > 57344
    return false;
  };
  std::vector<uint32_t> out(n);
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t p = 0;
    while (p < n_ladder && ladder[p] != schemes[i]) ++p;
    require(p < n_ladder, HR_EINVAL, "item " + std::to_string(i) + ": scheme not in the ladder");
    while (p > 0 && unsafe(ladder[p], stats[2 * i], (uint32_t)stats[2 * i + 1])) --p;
    out[i] = ladder[p];
  }
  return out;
}

}  // namespace harag
