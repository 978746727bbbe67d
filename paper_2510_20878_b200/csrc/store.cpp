// The HA-RAG store runtime (C++ / CUDA runtime API): packed chunk store,
// tier placement (Alg. 1 + Alg. 2 step 1 by bytes), request planning
// (Alg. 2 step 2 lookups), the host-tier streamer (pageable -> pinned bounce ->
// HBM staging ring) and epochs (hotness decay + re-placement).
#include "store.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <unordered_set>

#include "analysis.h"
#include "kernels.h"
#include "policy.h"
#include "trace.h"

namespace harag {

// ------------------------------------------------------------ FreeList
uint64_t FreeList::alloc(uint64_t size) {
  size = align_up(size, kAlign);
  for (auto it = free_.begin(); it != free_.end(); ++it) {  // first fit
    if (it->second >= size) {
      const uint64_t off = it->first, rest = it->second - size;
      free_.erase(it);
      if (rest) free_[off + size] = rest;
      used_ += size;
      return off;
    }
  }
  return kNone;
}

void FreeList::release(uint64_t off, uint64_t size) {
  size = align_up(size, kAlign);
  used_ -= size;
  auto it = free_.emplace(off, size).first;
  auto next = std::next(it);
  if (next != free_.end() && it->first + it->second == next->first) {
    it->second += next->second;
    free_.erase(next);
  }
  if (it != free_.begin()) {
    auto prev = std::prev(it);
    if (prev->first + prev->second == it->first) {
      prev->second += it->second;
      free_.erase(it);
    }
  }
}

// ---------------------------------------------------------------- Store
Store::Store(const hr_store_config& c) : cfg(c), lay(make_layout(c)) {
  require(cfg.n_ladder >= 1 && cfg.n_ladder <= 6, HR_EINVAL, "n_ladder must be 1..6");
  for (uint32_t j = 0; j < cfg.n_ladder; ++j) require(cfg.ladder[j] < HR_N_SCHEMES, HR_EINVAL, "unknown scheme in ladder");
  double sum = 0;
  for (uint32_t j = 0; j + 1 < cfg.n_ladder; ++j) {
    require(cfg.tau[j] >= 0.0 && cfg.tau[j] <= 1.0, HR_EINVAL, "tau out of [0,1]");
    sum += cfg.tau[j];
  }
  require(sum <= 1.0 + 1e-12, HR_EINVAL, "taus sum above 1");
  require(cfg.demand_mode == 0 || cfg.demand_mode == 1, HR_EINVAL, "demand_mode must be 0 or 1");
  if (cfg.demand_mode) cfg.keep_backing = 1;  // the backing plays the paper's disk: every item has a copy
  slots = cfg.staging_slots;  // 0: sized in ensure_ring once the largest item is known
  if (const char* g = std::getenv("HARAG_ASM_GRID")) grid_override = std::atoi(g);  // tuning experiments
  if (const char* g = std::getenv("HARAG_ASM_DYN")) asm_dyn_pct = (uint32_t)std::atoi(g);
  if (const char* g = std::getenv("HARAG_ASM_CHUNKS")) asm_dyn_per_cta = (uint32_t)std::atoi(g);
  HR_CUDA(cudaSetDevice(cfg.device));
  HR_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  if (cfg.numa_bind) local_cpus = gpu_local_cpus(cfg.device);
  host_prof = std::getenv("HARAG_HOST_PROF") != nullptr;
  if (const char* m = std::getenv("HARAG_METRICS_JSONL")) metrics = std::fopen(m, "a");  // per-call metrics
}

Store::~Store() {
  if (metrics) std::fclose(metrics);
  if (host_prof && prof_calls)
    std::fprintf(stderr, "[harag host prof] %llu calls, us/call: entry+validate %.2f desc_buffer %.2f pass1 %.2f "
                 "pass2-3 %.2f launchA %.2f tail %.2f\n", (unsigned long long)prof_calls,
                 1e3 * prof_ms[0] / prof_calls, 1e3 * prof_ms[1] / prof_calls, 1e3 * prof_ms[2] / prof_calls,
                 1e3 * prof_ms[3] / prof_calls, 1e3 * prof_ms[4] / prof_calls, 1e3 * prof_ms[5] / prof_calls);
  cudaSetDevice(cfg.device);
  cudaDeviceSynchronize();
  for (auto& d : dbuf) {
    if (d.dev) cudaFree(d.dev);
    if (d.host) cudaFreeHost(d.host);
    if (d.done) cudaEventDestroy(d.done);
  }
  for (uint8_t* b : bounce_rejects) cudaFreeHost(b);
  for (auto& r : ring) {
    if (r.dev) cudaFree(r.dev);
    if (r.bounce) cudaFreeHost(r.bounce);
    if (r.copied) cudaEventDestroy(r.copied);
    if (r.free_ev) cudaEventDestroy(r.free_ev);
  }
  for (auto& t : timers) cudaEventDestroy(t.first), cudaEventDestroy(t.second);
  for (auto& t : h2d_timers) cudaEventDestroy(t.first), cudaEventDestroy(t.second);
  for (auto& t : qtimers) cudaEventDestroy(t.first), cudaEventDestroy(t.second);
  copy_pool.reset();
  if (hbm_base) cudaFree(hbm_base);
  if (pin_base) cudaFreeHost(pin_base);
  if (page_base) free(page_base);
  if (backing_base) {
    if (backing_is_pinned)
      cudaFreeHost(backing_base);
    else
      free(backing_base);
  }
  if (delta) cudaFree(delta);
  if (att_part) cudaFree(att_part);
  if (att_done) cudaEventDestroy(att_done);
  if (asm_sched) cudaFree(asm_sched);
  if (att_cnt) cudaFree(att_cnt);
  if (err_flag) cudaFree(err_flag);
  if (scratch) cudaFree(scratch);
  if (gse_range) cudaFree(gse_range);
  if (src_k) cudaFree(src_k);
  if (src_v) cudaFree(src_v);
  if (start_ev) cudaEventDestroy(start_ev);
  if (after_a_ev) cudaEventDestroy(after_a_ev);
  for (auto& e : call_ev)
    if (e) cudaEventDestroy(e);
  if (mig_ev) cudaEventDestroy(mig_ev);
  for (auto& p : promos) cudaEventDestroy(p.ev);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (disk_fd >= 0) ::close(disk_fd);
  if (disk_fd_direct >= 0) ::close(disk_fd_direct);
}

uint32_t Store::logical_tier(uint32_t item) const {
  if (alg2)
    return alg2->contains(Alg2::GPU, item)    ? HR_T_HBM
           : alg2->contains(Alg2::PIN, item)  ? HR_T_PIN
           : alg2->contains(Alg2::PAGE, item) ? HR_T_PAGE
           : on_disk                          ? HR_T_DISK
                                              : HR_T_PAGE;
  return tier[item];  // eager: the placement target (a promotion may still be in flight)
}

uint8_t* Store::hbm_ptr(uint32_t item) const { return hbm_base + loc[item].hbm_off; }

// Pageable host memory for the backing / PAGE tier: 2 MiB aligned and advised as transparent huge pages
// (the boxes run THP in madvise mode): the bounce copies stream tens of GB through 4 KiB pages otherwise
// (HARAG_HOST_THP=0 keeps 4 KiB pages)
static uint8_t* alloc_pageable(uint64_t bytes) {
  constexpr uint64_t kHuge = 2ull << 20;
  const uint64_t n = (bytes + kHuge - 1) / kHuge * kHuge;
  uint8_t* p = (uint8_t*)aligned_alloc(kHuge, n);
  static const bool thp = !(std::getenv("HARAG_HOST_THP") && std::atoi(std::getenv("HARAG_HOST_THP")) == 0);
  if (p && thp) madvise(p, n, MADV_HUGEPAGE);  // advisory: failure leaves 4 KiB pages
  return p;
}

void Store::build_begin(uint32_t nd, const uint64_t* hot, const uint32_t* schemes) {
  require(state == State::Empty, HR_ESTATE, "store already built");
  require(nd > 0, HR_EINVAL, "n_docs must be > 0");
  require(hot != nullptr, HR_EINVAL, "hotness is NULL");
  if (schemes) {  // the caller's schemes (e.g. the value-distribution guard's), each one of the ladder
    for (uint32_t i = 0; i < 2 * nd; ++i)
      require(std::find(cfg.ladder, cfg.ladder + cfg.n_ladder, schemes[i]) != cfg.ladder + cfg.n_ladder, HR_EINVAL,
              "item " + std::to_string(i) + ": scheme not in the ladder");
    setup(nd, hot, std::vector<uint32_t>(schemes, schemes + 2 * nd), false);
  } else {
    // Alg. 1: schemes by hotness rank
    setup(nd, hot, assign_schemes(hot, 2 * nd, cfg.ladder, cfg.n_ladder, cfg.tau), false);
  }
  state = State::Building;
}

// Placement (Alg. 2 step 1 by bytes, R15) and every allocation of a store whose schemes are known.
// on_disk: the host backing of the cold items is the store file (hr_build_from_file, disk_backing).
std::vector<uint32_t> Store::place_lists() const {
  // pinned backing: every non-HBM item is served as PIN (no separate PIN_LIST); disk-backed stores add
  // a PAGE_LIST of page_budget bytes and leave the rest on disk (DISK_LIST)
  std::vector<uint32_t> t = lists_by_bytes(order, bytes.data(), cfg.hbm_budget,
                                           cfg.backing_pinned && !on_disk ? 0 : cfg.pin_budget,
                                           on_disk ? cfg.page_budget : ~0ull);
  return t;
}

void Store::setup(uint32_t nd, const uint64_t* hot, std::vector<uint32_t> sc, bool disk) {
  require(!disk || cfg.page_budget <= (1ull << 46), HR_EINVAL, "page_budget must be a finite byte count");
  const CpuBind bind(local_cpus);  // host tiers are allocated (and pinned pages touched) on the GPU's node
  on_disk = disk;
  HR_CUDA(cudaSetDevice(cfg.device));
  n_docs = nd;
  n_items = 2 * nd;
  h.assign(hot, hot + n_items);
  scheme = std::move(sc);
  bytes.resize(n_items);
  for (uint32_t i = 0; i < n_items; ++i) bytes[i] = lay.item_bytes(scheme[i]);
  // Alg. 2 step 1 by bytes (R15)
  order = rank_items(h.data(), n_items);
  tier = place_lists();
  if (cfg.demand_mode) {
    // Alg. 2 step 1 gives the lists; the queues start empty and fill on access (step 2)
    alg2.reset(new Alg2(n_items, tier.data(), bytes.data(), cfg.hbm_budget,
                        cfg.backing_pinned && !on_disk ? 0 : cfg.pin_budget, on_disk ? cfg.page_budget : 0));
    tier.assign(n_items, on_disk ? HR_T_DISK : HR_T_PAGE);
  } else if (cfg.backing_pinned && !on_disk) {
    for (auto& t : tier)
      if (t == HR_T_PAGE) t = HR_T_PIN;
  }
  loc.assign(n_items, Loc{});
  max_item = 0;
  for (uint32_t i = 0; i < n_items; ++i) max_item = std::max(max_item, bytes[i]);

  // HBM arena: the whole budget (re-placement may fill it differently later)
  if (cfg.hbm_budget) {
    uint64_t need = 0;
    for (uint32_t i = 0; i < n_items; ++i)
      if (tier[i] == HR_T_HBM) need += align_up(bytes[i], FreeList::kAlign);
    hbm_cap = cfg.keep_backing ? align_up(cfg.hbm_budget, FreeList::kAlign) : need;
    if (hbm_cap) {
      if (cudaMalloc(&hbm_base, hbm_cap) != cudaSuccess) {
        cudaGetLastError();
        fail(HR_ENOMEM, "cudaMalloc of the HBM arena failed");
      }
    }
    hbm.reset(hbm_cap);
  }
  // pageable PAGE tier cache (disk-backed stores)
  if (on_disk && cfg.page_budget) {
    page_cap = align_up(cfg.page_budget, FreeList::kAlign);
    page_base = alloc_pageable(page_cap);
    require(page_base != nullptr, HR_ENOMEM, "PAGE tier allocation failed");
    page.reset(page_cap);
  }
  // pinned tier (PIN_LIST copies when the backing is pageable or on disk)
  if ((!cfg.backing_pinned || on_disk) && cfg.pin_budget) {
    pin_cap = align_up(cfg.pin_budget, FreeList::kAlign);
    if (cudaHostAlloc((void**)&pin_base, pin_cap, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      fail(HR_ENOMEM, "cudaHostAlloc of the pinned tier failed");
    }
    pin.reset(pin_cap);
  }
  // host backing: one blob per item that needs one (all if keep_backing), aliased in bench mode
  uint64_t total = 0;
  std::map<uint64_t, uint64_t> alias_off;
  for (uint32_t i = 0; i < n_items && !disk; ++i) {
    if (!cfg.keep_backing && tier[i] == HR_T_HBM) continue;
    const uint64_t key = backing_key(i);
    auto it = alias_off.find(key);
    if (it != alias_off.end()) {
      loc[i].backing_off = it->second;
      loc[i].backing_alias = true;
    } else {
      loc[i].backing_off = total;
      alias_off[key] = total;
      total += align_up(bytes[i], 4096);
    }
  }
  if (total) {
    backing_is_pinned = cfg.backing_pinned != 0;
    if (backing_is_pinned) {
      if (cudaHostAlloc((void**)&backing_base, total, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        fail(HR_ENOMEM, "cudaHostAlloc of the pinned backing failed");
      }
    } else {
      backing_base = alloc_pageable(total);
      require(backing_base != nullptr, HR_ENOMEM, "host backing allocation failed");
    }
  }
  backing_bytes = total;
  // arena / pinned placement of the lists (eager mode)
  for (uint32_t pos = 0; pos < n_items && !cfg.demand_mode; ++pos) {
    const uint32_t i = order[pos];
    if (tier[i] == HR_T_HBM) {
      loc[i].hbm_off = hbm.alloc(bytes[i]);
      require(loc[i].hbm_off != FreeList::kNone, HR_ENOMEM, "HBM arena exhausted during placement");
    } else if (tier[i] == HR_T_PIN && pin_base) {
      loc[i].pin_off = pin.alloc(bytes[i]);
      require(loc[i].pin_off != FreeList::kNone, HR_ENOMEM, "pinned tier exhausted during placement");
    } else if (tier[i] == HR_T_PAGE && page_base) {
      loc[i].page_off = page.alloc(bytes[i]);
      require(loc[i].page_off != FreeList::kNone, HR_ENOMEM, "PAGE tier exhausted during placement");
    }
  }
  HR_CUDA(cudaMalloc(&delta, sizeof(int64_t) * n_items));
  HR_CUDA(cudaMemset(delta, 0, sizeof(int64_t) * n_items));
  HR_CUDA(cudaMalloc(&err_flag, sizeof(int)));
  HR_CUDA(cudaMemset(err_flag, 0, sizeof(int)));
  scratch = nullptr, scratch_items = 0;  // allocated by the first put that needs it
  HR_CUDA(cudaMalloc(&gse_range, sizeof(int) * 2 * 2 * kPutBatch * lay.n_slabs()));  // every item of a put batch
  put_done.assign(n_docs, 0);
  backing_filled.clear();
}

uint64_t Store::backing_key(uint32_t item) const {
  const uint32_t doc = item / 2, kind = item % 2;
  const uint32_t adoc = cfg.bench_alias_R ? doc % cfg.bench_alias_R : doc;
  if (!cfg.bench_alias_R) return item;
  return ((uint64_t)adoc * 2 + kind) * 8 + scheme[item];
}

void Store::build_put(uint32_t doc, const void* k_src, const void* v_src, cudaStream_t st) {
  build_put_batch(1, &doc, &k_src, &v_src, st);
}

void Store::build_put_batch(uint32_t n, const uint32_t* docs, const void* const* k_srcs, const void* const* v_srcs,
                            cudaStream_t st) {
  require(state == State::Building, HR_ESTATE, "hr_build_put outside begin/end");
  const CpuBind bind(local_cpus);  // the D2H fills first-touch the pageable backing pages
  require(n <= kPutBatch, HR_EINVAL, "hr_build_put_batch: at most 16 docs per call");
  require(n == 0 || (docs && k_srcs && v_srcs), HR_EINVAL, "NULL array");
  for (uint32_t i = 0; i < n; ++i) {
    require(docs[i] < n_docs, HR_ENOTFOUND, "doc id out of range");
    require(k_srcs[i] && v_srcs[i], HR_EINVAL, "source pointer is NULL");
    for (uint32_t j = 0; j < i; ++j) require(docs[j] != docs[i], HR_EINVAL, "duplicate doc in a put batch");
  }
  // items headed for the host only (not in the HBM arena) are quantised into scratch first
  uint32_t n_host = 0;
  for (uint32_t i = 0; i < 2 * n; ++i) n_host += tier[2 * docs[i / 2] + i % 2] != HR_T_HBM;
  if (n_host > scratch_items) {
    if (scratch) {  // a previous put may still be writing it
      HR_CUDA(cudaStreamSynchronize(st));
      cudaFree(scratch);
      scratch = nullptr;
    }
    HR_CUDA(cudaMalloc(&scratch, (size_t)n_host * max_item));
    scratch_items = n_host;
  }
  QuantParams q[2 * kPutBatch]{};
  uint8_t* dsts[2 * kPutBatch];
  uint32_t h = 0;
  for (uint32_t i = 0; i < 2 * n; ++i) {
    const uint32_t kind = i % 2, item = 2 * docs[i / 2] + kind;
    const uint32_t s = scheme[item];
    uint8_t* dst = tier[item] == HR_T_HBM ? hbm_ptr(item) : scratch + (size_t)(h++) * max_item;
    dsts[i] = dst;
    QuantParams& qk = q[i];
    qk.src = (const uint16_t*)(kind ? v_srcs[i / 2] : k_srcs[i / 2]);
    qk.dst = dst;
    qk.L = lay.L, qk.H = lay.H, qk.Hl = lay.Hl, qk.h0 = lay.h0, qk.T = lay.T, qk.D = lay.D, qk.G = lay.G;
    qk.gse_e = lay.gse_e, qk.gse_m = lay.gse_m, qk.dtype = lay.dtype, qk.scheme = s;
    qk.g_shift = (uint32_t)__builtin_ctz(lay.G);
    qk.code_bytes_slab = lay.code_bytes_slab(s);
    qk.meta_offset = lay.meta_offset(s);
    qk.meta_stride = lay.meta_stride(s);
    qk.err = err_flag;
    qk.gse_range = gse_range + (size_t)i * 2 * lay.n_slabs();
    // zero the padding (the kernels write codes and meta records only) so exported blobs are deterministic
    const uint64_t cend = lay.n_slabs() * qk.code_bytes_slab;
    const uint64_t mend = qk.meta_offset + lay.n_slabs() * qk.meta_stride;
    if (qk.meta_stride > lay.meta_raw_slab(s)) {  // padded records: zero the whole meta section
      HR_CUDA(cudaMemsetAsync(dst + cend, 0, bytes[item] - cend, st));
    } else {
      if (qk.meta_offset > cend) HR_CUDA(cudaMemsetAsync(dst + cend, 0, qk.meta_offset - cend, st));
      if (bytes[item] > mend) HR_CUDA(cudaMemsetAsync(dst + mend, 0, bytes[item] - mend, st));
    }
  }
  cudaEvent_t qa = nullptr, qb = nullptr;
  if (timing) {
    HR_CUDA(cudaEventCreate(&qa));
    HR_CUDA(cudaEventCreate(&qb));
    HR_CUDA(cudaEventRecord(qa, st));
  }
  launch_quantize(q, (int)(2 * n), st);
  if (timing) {
    HR_CUDA(cudaEventRecord(qb, st));
    qtimers.emplace_back(qa, qb);
  }
  for (uint32_t i = 0; i < 2 * n; ++i) {
    const uint32_t item = 2 * docs[i / 2] + i % 2;
    uint8_t* dst = dsts[i];
    if (loc[item].backing_off != FreeList::kNone && !backing_filled.count(loc[item].backing_off)) {
      // bench aliasing: a shared blob is written once (its docs have identical sources by contract)
      HR_CUDA(cudaMemcpyAsync(backing_base + loc[item].backing_off, dst, bytes[item], cudaMemcpyDeviceToHost, st));
      backing_filled.insert(loc[item].backing_off);
    }
    if (loc[item].pin_off != FreeList::kNone)
      HR_CUDA(cudaMemcpyAsync(pin_base + loc[item].pin_off, dst, bytes[item], cudaMemcpyDeviceToHost, st));
  }
  for (uint32_t i = 0; i < n; ++i) {
    if (!put_done[docs[i]]) ++n_put;
    put_done[docs[i]] = 1;
  }
}

void Store::build_end(cudaStream_t st) {
  require(state == State::Building, HR_ESTATE, "hr_build_end without hr_build_begin");
  HR_CUDA(cudaStreamSynchronize(st));
  int err = 0;
  HR_CUDA(cudaMemcpy(&err, err_flag, sizeof(int), cudaMemcpyDeviceToHost));
  require(n_put == n_docs, HR_EINVAL, "hr_build_end: not every doc was put");
  require(err == 0, HR_EINVAL, "NaN/Inf in the source chunks (rejected at ingestion, S:30)");
  cudaFree(scratch);
  scratch = nullptr;
  scratch_items = 0;
  state = State::Built;
}

void Store::build_with_source(uint32_t nd, const uint64_t* hot, hr_src_fn src, void* user, cudaStream_t st) {
  const NvtxRange nvtx_call("hr_build");
  require(src != nullptr, HR_EINVAL, "source callback is NULL");
  require(state == State::Empty, HR_ESTATE, "store already built");
  require(nd > 0 && hot != nullptr, HR_EINVAL, "n_docs must be > 0 and hotness non-NULL");
  // kSrcBatch docs per quantize launch: the source callback fills one buffer pair per doc
  const uint64_t full = 2ull * lay.L * lay.H * lay.T * lay.D;
  const uint32_t nb = std::max<uint32_t>(1, std::min<uint32_t>(kSrcBatch, nd));
  HR_CUDA(cudaSetDevice(cfg.device));
  HR_CUDA(cudaMalloc(&src_k, full * nb));
  HR_CUDA(cudaMalloc(&src_v, full * nb));
  if (cfg.guard) {
    // value-distribution guard (R29): a pass over every doc's source before placement, then Alg. 1's
    // schemes moved up the ladder where they would lose values
    const NvtxRange nvtx_guard("guard");
    unsigned long long* gs = nullptr;
    HR_CUDA(cudaMalloc((void**)&gs, sizeof(uint64_t) * 4ull * nd));
    HR_CUDA(cudaMemsetAsync(gs, 0, sizeof(uint64_t) * 4ull * nd, st));
    for (uint32_t doc = 0; doc < nd; ++doc) {
      const int rc = src(user, doc, src_k, src_v, (void*)st);
      require(rc == HR_OK, (hr_status)rc, "source callback failed for doc " + std::to_string(doc));
      launch_guard(lay.dtype, src_k, (uint64_t)lay.L * lay.H, lay.slab(), lay.gse_e, lay.gse_m, gs + 4ull * doc, st);
      launch_guard(lay.dtype, src_v, (uint64_t)lay.L * lay.H, lay.slab(), lay.gse_e, lay.gse_m, gs + 4ull * doc + 2,
                   st);
    }
    std::vector<uint64_t> stats(4ull * nd);
    HR_CUDA(cudaMemcpyAsync(stats.data(), gs, sizeof(uint64_t) * 4ull * nd, cudaMemcpyDeviceToHost, st));
    HR_CUDA(cudaStreamSynchronize(st));
    cudaFree(gs);
    const auto a1 = assign_schemes(hot, 2 * nd, cfg.ladder, cfg.n_ladder, cfg.tau);
    const auto sc = guard_schemes(a1.data(), stats.data(), 2 * nd, cfg.ladder, cfg.n_ladder);
    build_begin(nd, hot, sc.data());
  } else {
    build_begin(nd, hot);
  }
  uint32_t docs[kPutBatch];
  const void *ks[kPutBatch], *vs[kPutBatch];
  // bench aliasing (bench_alias_R > 0): a doc whose items all live only in a host backing blob that
  // an earlier doc with the same source already filled needs no quantisation (the blob would be
  // written with identical bytes) — only HBM-arena and pinned-tier items and first fills are built
  auto needed = [&](uint32_t doc) {
    if (!cfg.bench_alias_R) return true;
    for (uint32_t kind = 0; kind < 2; ++kind) {
      const Loc& l = loc[2 * doc + kind];
      if (tier[2 * doc + kind] == HR_T_HBM || l.pin_off != FreeList::kNone || l.page_off != FreeList::kNone ||
          l.backing_off == FreeList::kNone || !backing_filled.count(l.backing_off))
        return true;
    }
    return false;
  };
  uint32_t n = 0;
  auto flush = [&] {
    if (n) build_put_batch(n, docs, ks, vs, st);
    n = 0;
  };
  for (uint32_t doc = 0; doc < nd; ++doc) {
    if (!needed(doc)) {
      if (!put_done[doc]) ++n_put;
      put_done[doc] = 1;
      continue;
    }
    docs[n] = doc;
    ks[n] = (uint8_t*)src_k + full * n;
    vs[n] = (uint8_t*)src_v + full * n;
    const int rc = src(user, doc, (void*)ks[n], (void*)vs[n], (void*)st);
    require(rc == HR_OK, (hr_status)rc, "source callback failed for doc " + std::to_string(doc));
    if (++n == nb) flush();
  }
  flush();
  build_end(st);
  cudaFree(src_k);
  cudaFree(src_v);
  src_k = src_v = nullptr;
}

// --------------------------------------------------------------- assemble
Store::DescBuf& Store::desc_buffer(size_t n) {
  if (dbuf.empty()) dbuf.resize(kDescBufs);
  DescBuf& d = dbuf[dbuf_next];
  dbuf_next = (dbuf_next + 1) % kDescBufs;
  if (d.done) HR_CUDA(cudaEventSynchronize(d.done));  // previous user of this buffer finished
  else HR_CUDA(cudaEventCreateWithFlags(&d.done, cudaEventDisableTiming));
  if (d.cap < n) {
    if (d.dev) HR_CUDA(cudaFree(d.dev));
    if (d.host) HR_CUDA(cudaFreeHost(d.host));
    d.cap = std::max<size_t>(n, 256);
    HR_CUDA(cudaMalloc(&d.dev, d.cap * sizeof(AsmDesc)));
    HR_CUDA(cudaHostAlloc((void**)&d.host, d.cap * sizeof(AsmDesc), cudaHostAllocPortable));
  }
  return d;
}

#ifndef HARAG_MAX_SLOTS
#define HARAG_MAX_SLOTS 128
#endif
// At most this many staging slots: a call that streams more host-tier items than there are slots reuses a
// slot within the call, and that copy then waits for the slot's launch B, which runs behind launch A
// (the copy stream idles for launch A's ~4.5 ms at C2 batch 32).  128 covers C2's ~58 items per call with
// its Zipf spread: link fraction in the copy window 0.936 -> 0.983 (pinned), 0.91 -> 0.95-0.97 (pageable).
constexpr uint64_t kMaxSlots = HARAG_MAX_SLOTS;

void Store::ensure_ring() {
  if (!ring.empty()) return;
  // Default depth: ~2 GiB of slots (3..64).  Launch B of a streamed item runs on the request stream
  // behind launch A, so a slot is recycled only after launch A; the ring must hold what the link
  // delivers meanwhile (Llama-3-8B batch 32: launch A ~5 ms = ~280 MB at 55 GB/s) or the copies stall.
  if (!slots) slots = (uint32_t)std::min<uint64_t>(kMaxSlots, std::max<uint64_t>(3, ((2ull << 30) + max_item - 1) / max_item));
  ring.resize(slots);
  for (auto& r : ring) {
    HR_CUDA(cudaMalloc(&r.dev, max_item));
    HR_CUDA(cudaEventCreateWithFlags(&r.copied, cudaEventDisableTiming));
    HR_CUDA(cudaEventCreateWithFlags(&r.free_ev, cudaEventDisableTiming));
  }
}

// The pinned bounce buffers of every ring slot, allocated on first need and each probed with timed H2D
// copies (best of 2) into a scratch device buffer: the physical placement of freshly pinned pages varies
// and a slow buffer slows every item routed through its slot (tools/pin_probe.py on the 16-vCPU B200
// host: most 16 MiB buffers 54.3 GB/s, one or two of 16 at 29-43 GB/s, the pageable leg bimodal 0.6 /
// 0.9 of the link per process).  A buffer below 90% of the fastest probe is replaced (up to 4 times per
// slot, at most 2 x slots rejects in all) and kept pinned until the store closes, so the allocator cannot
// hand the same pages back.
void Store::ensure_bounce(Slot& first) {
  if (first.bounce) return;
  const size_t n = align_up(max_item, 4096);
  cudaEvent_t e0, e1;
  HR_CUDA(cudaEventCreate(&e0));
  HR_CUDA(cudaEventCreate(&e1));
  uint8_t* dev = nullptr;  // a scratch destination: the slots' device buffers may hold items in flight
  HR_CUDA(cudaMalloc(&dev, n));
  auto probe = [&](uint8_t* buf) {
    float best = 1e30f;
    for (int rep = 0; rep < 2; ++rep) {
      HR_CUDA(cudaEventRecord(e0, copy_stream));
      HR_CUDA(cudaMemcpyAsync(dev, buf, n, cudaMemcpyHostToDevice, copy_stream));
      HR_CUDA(cudaEventRecord(e1, copy_stream));
      HR_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      HR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    return (double)n / (best * 1e-3) / 1e9;
  };
  HR_CUDA(cudaStreamSynchronize(copy_stream));  // earlier copies of this call finish first (first use only)
  for (auto& sl : ring) {
    if (sl.bounce) continue;
    for (int attempt = 0;; ++attempt) {
      uint8_t* b = nullptr;
      HR_CUDA(cudaHostAlloc((void**)&b, n, cudaHostAllocPortable));
      const double gbps = probe(b);
      bounce_best_gbps = std::max(bounce_best_gbps, gbps);
      if (gbps >= 0.9 * bounce_best_gbps || attempt == 4 || bounce_rejects.size() >= 2 * ring.size()) {
        sl.bounce = b;
        break;
      }
      bounce_rejects.push_back(b);
    }
  }
  // a buffer accepted before a faster probe raised the bar: re-check once against the final best
  for (auto& sl : ring) {
    if (probe(sl.bounce) >= 0.9 * bounce_best_gbps) continue;
    for (int attempt = 0; attempt < 4 && bounce_rejects.size() < 2 * ring.size(); ++attempt) {
      uint8_t* b = nullptr;
      HR_CUDA(cudaHostAlloc((void**)&b, n, cudaHostAllocPortable));
      if (probe(b) >= 0.9 * bounce_best_gbps) {
        bounce_rejects.push_back(sl.bounce);
        sl.bounce = b;
        break;
      }
      bounce_rejects.push_back(b);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dev);
}

void Store::launch(const AsmDesc* dev_descs, const AsmDesc* host_descs, uint32_t n, uint32_t k, uint32_t scheme_mask,
                   cudaStream_t st) {
  AsmParams p{};
  p.n_desc = n;
  if (n <= (uint32_t)kAsmInline) {  // carried in the kernel parameters: no descriptor copy ahead of the launch
    p.descs = nullptr;
    std::memcpy(p.inl, host_descs, n * sizeof(AsmDesc));
  } else {
    p.descs = dev_descs;
  }
  p.L = lay.L, p.Hl = lay.Hl, p.T = lay.T, p.D = lay.D, p.k = k, p.G = lay.G;
  p.g_shift = (uint32_t)__builtin_ctz(lay.G);
  p.gse_m = lay.gse_m;
  p.dtype = lay.dtype;
  p.slab = (uint32_t)lay.slab();
  for (uint32_t s = 0; s < HR_N_SCHEMES; ++s) p.meta_stride[s] = (uint32_t)lay.meta_stride(s);
  if (asm_dyn_pct) {
    if (!asm_sched) {
      HR_CUDA(cudaMalloc((void**)&asm_sched, 64 * 16));
      HR_CUDA(cudaMemset(asm_sched, 0, 64 * 16));
    }
    p.sched = asm_sched + 4 * (asm_sched_next++ % 64);
    p.dyn_pct = asm_dyn_pct;
    p.dyn_per_cta = asm_dyn_per_cta;
  }
  cudaEvent_t a = nullptr, b = nullptr;
  if (timing) {
    HR_CUDA(cudaEventCreate(&a));
    HR_CUDA(cudaEventCreate(&b));
    HR_CUDA(cudaEventRecord(a, st));
  }
  launch_assemble(p, scheme_mask, st, grid_override);
  if (timing) {
    HR_CUDA(cudaEventRecord(b, st));
    timers.emplace_back(a, b);
  }
  stats.kernel_launches++;
}

void Store::validate_request(uint32_t n_req, uint32_t k, const uint32_t* ids, void* const* k_out,
                             void* const* v_out) const {
  require(state == State::Built, HR_ESTATE, "hr_assemble_kv before the store is built");
  require(n_req > 0 && k > 0, HR_EINVAL, "n_req and k must be > 0");
  require(ids && k_out && v_out, HR_EINVAL, "NULL argument");
  uint32_t stack_ids[64];  // k <= 64 in practice: no heap allocation per call
  std::vector<uint32_t> heap_ids(k > 64 ? k : 0);
  uint32_t* tmp = k > 64 ? heap_ids.data() : stack_ids;
  for (uint32_t r = 0; r < n_req; ++r) {
    require(k_out[r] && v_out[r], HR_EINVAL, "NULL output pointer");
    require(((uintptr_t)k_out[r] & 15) == 0 && ((uintptr_t)v_out[r] & 15) == 0, HR_EINVAL,
            "output pointers must be 16-byte aligned");
    for (uint32_t j = 0; j < k; ++j) {
      tmp[j] = ids[(uint64_t)r * k + j];
      if (tmp[j] >= n_docs) fail(HR_ENOTFOUND, "unknown doc id " + std::to_string(tmp[j]));
    }
    std::sort(tmp, tmp + k);
    if (std::adjacent_find(tmp, tmp + k) != tmp + k)
      fail(HR_EINVAL, "duplicate doc id in request " + std::to_string(r) + " (R19)");
  }
}

// Demand mode (paper-literal Alg. 2 step 2): pinned / pageable space freed by evictions of the
// previous call is released now — the copy stream is drained before pinned space is rewritten by
// the host.  (HBM arena space is released inside the call that evicts; promotion copies are
// ordered after its readers by `start_ev` and `after_a_ev`.)
void Store::release_deferred() {
  if (!pending_pin_free.empty()) {
    HR_CUDA(cudaStreamSynchronize(copy_stream));
    for (auto& f : pending_pin_free) pin.release(f.first, f.second);
    pending_pin_free.clear();
  }
  for (auto& f : pending_page_free) page.release(f.first, f.second);  // read by the host during its call
  pending_page_free.clear();
}

void Store::assemble(uint32_t n_req, uint32_t k, const uint32_t* ids, void* const* k_out, void* const* v_out,
                     cudaStream_t st) {
  const auto host_t0 = std::chrono::steady_clock::now();
  const NvtxRange nvtx_call("hr_assemble_kv");
  const hr_stats before = metrics ? stats : hr_stats{};
  auto tick = [&](int i) {
    if (!host_prof) return;
    const auto now = std::chrono::steady_clock::now();
    prof_ms[i] += std::chrono::duration<double, std::milli>(now - prof_t).count();
    prof_t = now;
  };
  if (host_prof) prof_t = host_t0;
  validate_request(n_req, k, ids, k_out, v_out);  // before any device work: no partial writes
  HR_CUDA(cudaSetDevice(cfg.device));
  if (call_timing) {  // per-call latency: this event -> the end of the call's last launch (device clock)
    if (!call_ev[0]) {
      HR_CUDA(cudaEventCreate(&call_ev[0]));
      HR_CUDA(cudaEventCreate(&call_ev[1]));
    }
    HR_CUDA(cudaEventRecord(call_ev[0], st));
  }
  tick(0);
  if (!promos.empty()) poll_promotions(false);
  const bool demand = alg2 != nullptr;
  if (demand) {
    release_deferred();
    if (!start_ev) HR_CUDA(cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming));
    HR_CUDA(cudaEventRecord(start_ev, st));  // every kernel that may read freed arena space
    HR_CUDA(cudaStreamWaitEvent(copy_stream, start_ev, 0));
  }
  const size_t n_desc = 2ull * n_req * k;
  if (hdesc.size() < n_desc) hdesc.resize(n_desc);  // host descriptors (pageable scratch)
  tick(1);
  std::optional<NvtxRange> nvtx_plan(std::in_place, "plan");
  // a6 planning, in three passes.
  //  1. Every access in request order: Alg. 2 step 2 (demand mode: one branch per access, the hit
  //     counted where Alg. 2 finds the item, host-queue fills done at once) or the tier lookup (eager).
  //  2. Demand mode: physical HBM residency := queueGPU as it stands after the call's accesses.
  //     Blocks of items that left the queue are freed first (their launch-A readers of this call are
  //     ordered before any promotion copy that reuses the space: `after_a`), then the newcomers that
  //     this call accessed get their arena blocks; their DMA lands there instead of a ring slot.
  //  3. Descriptors: items resident when the call started go to launch A (from their block as it was
  //     at the start), the rest are streamed, each item once per call.
  std::vector<uint32_t> evicted_gpu;
  for (uint32_t r = 0; r < n_req; ++r) {
    for (uint32_t j = 0; j < k; ++j) {
      for (uint32_t kind = 0; kind < 2; ++kind) {
        const uint32_t item = 2 * ids[(uint64_t)r * k + j] + kind;
        stats.bytes_out += lay.n_slabs() * lay.slab() * 2;
        stats.bytes_hbm_alg += lay.n_slabs() * lay.slab() * 2 + bytes_read_alg(item);
        if (demand) {  // Alg. 2 step 2: one branch per access, inclusive promotion, LRU
          const Alg2::Outcome o = alg2->access(item);
          if (o.hit == Alg2::DISK && on_disk)
            stats.hits_disk++;
          else
            stats.hits[o.hit == Alg2::GPU ? HR_T_HBM : o.hit == Alg2::PIN ? HR_T_PIN : HR_T_PAGE]++;
          for (const auto& ev : o.evicted) {
            Loc& l = loc[ev.second];
            if (ev.first == Alg2::GPU) {
              evicted_gpu.push_back(ev.second);  // pass 2 frees its block unless it is back in the queue
            } else if (ev.first == Alg2::PIN && l.pin_off != FreeList::kNone) {
              pending_pin_free.emplace_back(l.pin_off, bytes[ev.second]);
              l.pin_off = FreeList::kNone;
            } else if (ev.first == Alg2::PAGE && l.page_off != FreeList::kNone) {
              pending_page_free.emplace_back(l.page_off, bytes[ev.second]);
              l.page_off = FreeList::kNone;
            }
          }
          if ((o.put_mask & (1u << Alg2::PAGE)) && loc[item].page_off == FreeList::kNone && page_base) {
            const uint64_t off = page.alloc(bytes[item]);  // queuePAGE.put: a pageable copy from disk
            if (off != FreeList::kNone) {
              loc[item].page_off = off;
              fill_host(item, page_base + off);
            }
          }
          if ((o.put_mask & (1u << Alg2::PIN)) && loc[item].pin_off == FreeList::kNone && pin_base) {
            const uint64_t off = pin.alloc(bytes[item]);  // queuePIN.put: a pinned copy from the backing
            if (off != FreeList::kNone) {
              loc[item].pin_off = off;
              fill_host(item, pin_base + off);
            }
          }
        } else {
          const Loc& l = loc[item];
          if (l.hbm_off == FreeList::kNone && l.pin_off == FreeList::kNone && l.page_off == FreeList::kNone &&
              l.backing_off == FreeList::kNone)
            stats.hits_disk++;
          else
            stats.hits[l.hbm_off != FreeList::kNone                                                    ? HR_T_HBM
                       : (l.pin_off != FreeList::kNone || (l.backing_off != FreeList::kNone && backing_is_pinned &&
                                                          l.page_off == FreeList::kNone)) ? HR_T_PIN
                                                                                           : HR_T_PAGE]++;
        }
      }
    }
  }
  // pass 2 (demand mode): HBM arena := queueGPU
  tick(2);
  std::unordered_map<uint32_t, uint64_t> start_off;  // items resident at the call's start whose block was freed
  std::unordered_map<uint32_t, bool> promoted;       // item -> its arena block reuses space freed in this call
  if (demand) {
    std::vector<std::pair<uint64_t, uint64_t>> freed;  // [off, off + size) freed in this call
    for (uint32_t item : evicted_gpu) {
      Loc& l = loc[item];
      if (l.hbm_off == FreeList::kNone || alg2->contains(Alg2::GPU, item)) continue;
      start_off.emplace(item, l.hbm_off);
      freed.emplace_back(l.hbm_off, l.hbm_off + align_up(bytes[item], FreeList::kAlign));
      hbm.release(l.hbm_off, bytes[item]);
      l.hbm_off = FreeList::kNone;
      stats.migrations_out++;
    }
    for (uint64_t a = 0; a < 2ull * n_req * k; ++a) {
      const uint32_t item = 2 * ids[a / 2] + (uint32_t)(a % 2);
      if (loc[item].hbm_off != FreeList::kNone || !alg2->contains(Alg2::GPU, item)) continue;
      uint64_t off = hbm.alloc(bytes[item]);
      if (off == FreeList::kNone && hbm_cap - hbm.used() >= align_up(bytes[item], FreeList::kAlign)) {
        // queueGPU fits the budget by construction: defragment (needs an idle device) and retry.  The
        // moved blocks overwrite the space of items freed above, so those are streamed instead.
        HR_CUDA(cudaDeviceSynchronize());
        compact_hbm();
        start_off.clear();
        freed.clear();
        for (auto& p : promoted) p.second = false;
        off = hbm.alloc(bytes[item]);
      }
      if (off == FreeList::kNone) {
        stats.failed_promotions++;
        continue;
      }
      bool reuse = false;
      const uint64_t end = off + align_up(bytes[item], FreeList::kAlign);
      for (const auto& f : freed) reuse |= off < f.second && f.first < end;
      loc[item].hbm_off = off;  // "put C_i in queueGPU": resident once its copy (ordered below) lands
      promoted.emplace(item, reuse);
      stats.migrations_in++;
    }
  }
  // pass 3: descriptors
  struct Stream {
    uint32_t item;
    uint64_t arena_off;  // != kNone: promotion target (demand mode), else a staging-ring slot
    bool after_a;        // the arena block reuses space a launch-A descriptor of this call reads
    std::vector<AsmDesc> descs;
  };
  std::vector<Stream> streamed;
  std::unordered_map<uint32_t, size_t> stream_idx;
  size_t nh = 0;
  uint32_t hbm_mask = 0;
  bool any_after_a = false;
  for (uint32_t r = 0; r < n_req; ++r) {
    const bool counted = ((req_counter + r) % (uint64_t)cfg.world) == (uint64_t)cfg.rank;
    for (uint32_t j = 0; j < k; ++j) {
      for (uint32_t kind = 0; kind < 2; ++kind) {
        const uint32_t item = 2 * ids[(uint64_t)r * k + j] + kind;
        AsmDesc d{};
        d.out = (uint8_t*)(kind ? v_out[r] : k_out[r]);
        d.count = counted ? reinterpret_cast<unsigned long long*>(delta + item) : nullptr;
        d.slot = j;
        d.scheme = scheme[item];
        const auto pr = promoted.find(item);
        const auto so = start_off.find(item);
        if (pr == promoted.end() && (loc[item].hbm_off != FreeList::kNone || so != start_off.end())) {
          d.codes = hbm_base + (so != start_off.end() ? so->second : loc[item].hbm_off);
          d.meta = d.codes + lay.meta_offset(d.scheme);
          hdesc[nh++] = d;
          hbm_mask |= 1u << d.scheme;
          continue;
        }
        auto it = stream_idx.find(item);
        if (it == stream_idx.end()) {
          Stream s{item, FreeList::kNone, false, {}};
          if (pr != promoted.end()) {
            s.arena_off = loc[item].hbm_off;
            s.after_a = pr->second;
            any_after_a |= pr->second;
          }
          it = stream_idx.emplace(item, streamed.size()).first;
          streamed.push_back(std::move(s));
        }
        streamed[it->second].descs.push_back(d);
      }
    }
  }
  // descriptors of streamed items point at their arena slot or staging-ring slot
  if (!streamed.empty()) ensure_ring();
  size_t pos = nh, ring_i = 0;
  std::vector<uint8_t*> dest(streamed.size());
  std::vector<std::pair<size_t, size_t>> range(streamed.size());
  for (size_t i = 0; i < streamed.size(); ++i) {
    Stream& s = streamed[i];
    dest[i] = s.arena_off != FreeList::kNone ? hbm_base + s.arena_off : ring[ring_i++ % slots].dev;
    const size_t b = pos;
    for (AsmDesc d : s.descs) {
      d.codes = dest[i];
      d.meta = dest[i] + lay.meta_offset(d.scheme);
      hdesc[pos++] = d;
    }
    range[i] = {b, pos - b};
  }
  tick(3);
  nvtx_plan.reset();
  bool need_dev = nh > (size_t)kAsmInline;
  for (const auto& rg : range) need_dev |= rg.second > (size_t)kAsmInline;
  // launches of <= kAsmInline descriptors carry them as kernel parameters; only larger ones need the
  // device array (a pinned staging buffer, recycled once the call's launches are done)
  DescBuf* db = nullptr;
  const AsmDesc* ddesc = nullptr;
  if (need_dev) {
    db = &desc_buffer(pos);
    std::memcpy(db->host, hdesc.data(), pos * sizeof(AsmDesc));
    HR_CUDA(cudaMemcpyAsync(db->dev, db->host, pos * sizeof(AsmDesc), cudaMemcpyHostToDevice, st));
    ddesc = db->dev;
  }
  // launch A: every resident (request, slot, kind)
  if (nh) {
    const NvtxRange r("launch_a");
    launch(ddesc, hdesc.data(), (uint32_t)nh, k, hbm_mask, st);
  }
  tick(4);
  if (any_after_a && nh) {
    if (!after_a_ev) HR_CUDA(cudaEventCreateWithFlags(&after_a_ev, cudaEventDisableTiming));
    HR_CUDA(cudaEventRecord(after_a_ev, st));
  }
  // a7: host-tier items -> (pinned, or pageable -> pinned bounce) -> HBM (ring slot or arena) -> launch B
  cudaEvent_t c0 = nullptr, c1 = nullptr;
  if (timing && !streamed.empty()) {
    HR_CUDA(cudaEventCreate(&c0));
    HR_CUDA(cudaEventCreate(&c1));
  }
  ring_i = 0;
  std::optional<NvtxRange> nvtx_stream;
  if (!streamed.empty()) nvtx_stream.emplace("host_tier_stream");
  for (size_t i = 0; i < streamed.size(); ++i) {
    const uint32_t item = streamed[i].item;
    const bool to_arena = streamed[i].arena_off != FreeList::kNone;
    Slot& sl = ring[(to_arena ? ring_i : ring_i++) % slots];
    const uint8_t* src = nullptr;
    bool bounce = false, from_disk = false;
    if (loc[item].pin_off != FreeList::kNone) {
      src = pin_base + loc[item].pin_off;
    } else if (loc[item].page_off != FreeList::kNone) {
      src = page_base + loc[item].page_off;  // PAGE tier: pageable, through the bounce
      bounce = true;
    } else if (loc[item].backing_off != FreeList::kNone) {
      src = backing_base + loc[item].backing_off;
      bounce = !backing_is_pinned;
    } else {
      from_disk = true;  // the DISK tier ("load C_i from Disk"): file -> pinned bounce -> HBM
    }
    if (!to_arena) HR_CUDA(cudaStreamWaitEvent(copy_stream, sl.free_ev, 0));
    if (to_arena && streamed[i].after_a && nh) HR_CUDA(cudaStreamWaitEvent(copy_stream, after_a_ev, 0));
    if (c0 && i == 0) HR_CUDA(cudaEventRecord(c0, copy_stream));
    if (from_disk) {
      ensure_bounce(sl);
      if (sl.used) HR_CUDA(cudaEventSynchronize(sl.copied));
      read_disk(item, sl.bounce);
      HR_CUDA(cudaMemcpyAsync(dest[i], sl.bounce, bytes[item], cudaMemcpyHostToDevice, copy_stream));
    } else if (bounce) {
      // pageable data is first copied to pinned memory (non-temporal stores, every host core).
      // Whole-item pieces by default: the copy of item i+1 overlaps the DMA of item i, and splitting an
      // item over the pool in smaller pieces measured slower (tools/bounce_bench.cpp: 2 / 4 / 8 MiB /
      // whole 16.5 MiB pieces on 16 threads: 23 / 32 / 30 / 43 GB/s).
      ensure_bounce(sl);
      if (sl.used) HR_CUDA(cudaEventSynchronize(sl.copied));  // previous DMA out of this bounce buffer done
      static const size_t kPiece = std::getenv("HARAG_BOUNCE_PIECE") ? (size_t)std::atoll(std::getenv("HARAG_BOUNCE_PIECE"))
                                                                    : (size_t)1 << 40;
      const NvtxRange r("bounce");
      for (size_t off = 0; off < bytes[item]; off += kPiece) {
        const size_t n = std::min<size_t>(kPiece, bytes[item] - off);
        host_copy(sl.bounce + off, src + off, n);
        HR_CUDA(cudaMemcpyAsync(dest[i] + off, sl.bounce + off, n, cudaMemcpyHostToDevice, copy_stream));
      }
    } else {
      HR_CUDA(cudaMemcpyAsync(dest[i], src, bytes[item], cudaMemcpyHostToDevice, copy_stream));
    }
    HR_CUDA(cudaEventRecord(sl.copied, copy_stream));
    if (c1 && i + 1 == streamed.size()) {
      HR_CUDA(cudaEventRecord(c1, copy_stream));
      h2d_timers.emplace_back(c0, c1);
    }
    stats.h2d_items++;
    sl.used = true;
    stats.bytes_h2d += bytes[item];
    HR_CUDA(cudaStreamWaitEvent(st, sl.copied, 0));
    {
      const NvtxRange r("launch_b");
      launch(ddesc ? ddesc + range[i].first : nullptr, hdesc.data() + range[i].first, (uint32_t)range[i].second, k,
             1u << scheme[item], st);
    }
    if (!to_arena) HR_CUDA(cudaEventRecord(sl.free_ev, st));
  }
  nvtx_stream.reset();
  if (db) HR_CUDA(cudaEventRecord(db->done, st));
  if (call_timing) {
    HR_CUDA(cudaEventRecord(call_ev[1], st));
    call_recorded = true;
  }
  tick(5);
  prof_calls++;
  const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
  stats.host_ms += host_ms;
  req_counter += n_req;
  stats.requests += n_req;
  if (metrics) {  // HARAG_METRICS_JSONL: one line per call (host-side counters, no device synchronisation)
    std::fprintf(metrics,
                 "{\"call\": %llu, \"n_req\": %u, \"k\": %u, \"hits\": [%llu, %llu, %llu], \"hits_disk\": %llu, "
                 "\"bytes_out\": %llu, \"bytes_h2d\": %llu, \"h2d_items\": %llu, \"launches\": %llu, "
                 "\"host_us\": %.2f}\n",
                 (unsigned long long)metrics_calls++, n_req, k,
                 (unsigned long long)(stats.hits[0] - before.hits[0]), (unsigned long long)(stats.hits[1] - before.hits[1]),
                 (unsigned long long)(stats.hits[2] - before.hits[2]),
                 (unsigned long long)(stats.hits_disk - before.hits_disk),
                 (unsigned long long)(stats.bytes_out - before.bytes_out),
                 (unsigned long long)(stats.bytes_h2d - before.bytes_h2d),
                 (unsigned long long)(stats.h2d_items - before.h2d_items),
                 (unsigned long long)(stats.kernel_launches - before.kernel_launches), 1e3 * host_ms);
  }
}

double Store::last_call_ms() {
  require(call_recorded, HR_ESTATE, "no timed hr_assemble_kv call (hr_set_timing bit 1)");
  HR_CUDA(cudaEventSynchronize(call_ev[1]));
  float ms = 0;
  HR_CUDA(cudaEventElapsedTime(&ms, call_ev[0], call_ev[1]));
  return ms;
}

// A host copy of item's blob at dst (pinned-tier fill): from the in-memory backing or the store file.
void Store::fill_host(uint32_t item, uint8_t* dst) {
  if (loc[item].backing_off != FreeList::kNone) {
    host_copy(dst, backing_base + loc[item].backing_off, bytes[item]);
  } else {
    require(disk_fd >= 0, HR_ESTATE, "item has no host copy");
    uint64_t done = 0;
    while (done < bytes[item]) {
      const ssize_t r = ::pread(disk_fd, dst + done, bytes[item] - done, (off_t)(disk_off[item] + done));
      require(r > 0, HR_EINVAL, "read " + disk_path + ": " + std::strerror(errno));
      done += (uint64_t)r;
    }
  }
}

void Store::host_copy(void* dst, const void* src, size_t n) {
  if (!copy_pool) {
    // half the host cores (+ the calling thread): the bounce copies share host DRAM with the DMA they
    // feed, so more copy threads starve the link (tools/bounce_bench.cpp on the 16-core B200 host, whole
    // 16.5 MiB items, non-temporal stores, 3 runs each: 7 workers 45.4-45.8 GB/s on the link, 9 workers
    // 50.5-51.2, 11 workers 48.1-48.8, 15 workers 44.1-46.8; pinned DMA alone 54.8)
    unsigned t = std::max(1u, std::thread::hardware_concurrency()) / 2 + 1;
    if (const char* e = std::getenv("HARAG_COPY_THREADS")) t = (unsigned)std::atoi(e);
    const int spin = std::getenv("HARAG_POOL_SPIN") ? std::atoi(std::getenv("HARAG_POOL_SPIN")) : 2000;
    const bool nt = !(std::getenv("HARAG_COPY_NT") && std::atoi(std::getenv("HARAG_COPY_NT")) == 0);
    copy_pool.reset(new CopyPool(std::min(t, 31u), spin, nt));
    copy_pool->set_affinity(local_cpus);
  }
  if (n) copy_pool->copy(dst, src, n);
}

uint64_t Store::bytes_read_alg(uint32_t item) const {
  const uint32_t s = scheme[item];
  return lay.n_slabs() * (lay.code_bytes_slab(s) + lay.meta_raw_slab(s));
}

// ---------------------------------------------------------------- epochs
void Store::poll_promotions(bool wait_all) {
  size_t w = 0;
  for (auto& p : promos) {
    const cudaError_t q = wait_all ? cudaEventSynchronize(p.ev) : cudaEventQuery(p.ev);
    if (q == cudaSuccess) {
      loc[p.item].hbm_off = p.off;  // the copy landed: served from HBM from now on
      cudaEventDestroy(p.ev);
    } else if (q == cudaErrorNotReady) {
      promos[w++] = p;
    } else {
      HR_CUDA(q);
    }
  }
  promos.resize(w);
}

// a9 re-placement.  Eviction frees arena space at once: the promotion copies that may reuse it are
// ordered (copy stream waits `mig_ev`) after every launch already enqueued on `st`, and no later
// launch reads an evicted item from HBM.  Promotions are asynchronous: an item becomes resident
// when its copy event has completed (polled at the next hr_assemble_kv), and until then it is
// streamed from the host like any host-tier item — requests never wait for a migration.
// Consumer: attention over the request's packed chunks (kernels/attend.cu), for
// the layer window [l0, l0 + nl).  HBM-resident items are read in place; every other item is staged
// first: the window's code and meta slabs (contiguous runs of the blob) are copied from
// the pinned tier / host backing (pageable through the pinned bounce; disk through a read of
// the blob) into a staging-ring slot, and the launch waits for those copies.  A call's host-tier
// items must fit the ring at once (HR_ESTATE otherwise, before any work).
void Store::attend(uint32_t n_req, uint32_t k, const uint32_t* ids, uint32_t l0, uint32_t nl, const void* q,
                   uint32_t n_q, uint32_t g, void* o, float* lse, float scale, void* kv_dump, cudaStream_t st,
                   const void* k_own, const void* v_own) {
  const NvtxRange nvtx_call("hr_attend");
  require(state == State::Built, HR_ESTATE, "hr_attend before the store is built");
  require(!alg2, HR_ESTATE, "hr_attend needs eager placement (demand_mode = 0)");
  require(q && o, HR_EINVAL, "NULL query or output pointer");
  require(((uintptr_t)q & 15) == 0 && ((uintptr_t)o & 15) == 0 && ((uintptr_t)kv_dump & 15) == 0, HR_EINVAL,
          "query / output pointers must be 16-byte aligned");
  require((k_own == nullptr) == (v_own == nullptr), HR_EINVAL, "own K and V go together");
  require(((uintptr_t)k_own & 15) == 0 && ((uintptr_t)v_own & 15) == 0, HR_EINVAL,
          "own K / V pointers must be 16-byte aligned");
  require(!k_own || (n_q <= 64 && k <= 63), HR_EINVAL, "prefill form: n_q <= 64 question tokens and k <= 63");
  require(g >= 1 && n_q >= 1 && (uint64_t)g * n_q <= 128, HR_EINVAL, "g * n_q must be in [1, 128]");
  require(lay.D == 64 || lay.D == 128, HR_EINVAL, "hr_attend: head_dim must be 64 or 128");
  require(lay.T % 64 == 0, HR_EINVAL, "hr_attend: tokens per chunk must be a multiple of 64");
  require(nl >= 1 && l0 < lay.L && nl <= lay.L - l0, HR_EINVAL, "hr_attend: layer window outside [0, L)");
  require(n_req == 0 || (k >= 1 && ids), HR_EINVAL, "bad request");
  std::vector<uint32_t> tmp(k);
  for (uint32_t r = 0; r < n_req; ++r) {
    for (uint32_t j = 0; j < k; ++j) {
      tmp[j] = ids[(uint64_t)r * k + j];
      if (tmp[j] >= n_docs) fail(HR_ENOTFOUND, "unknown doc id " + std::to_string(tmp[j]));
    }
    std::sort(tmp.begin(), tmp.end());
    if (std::adjacent_find(tmp.begin(), tmp.end()) != tmp.end())
      fail(HR_EINVAL, "duplicate doc id in request " + std::to_string(r) + " (R19)");
  }
  HR_CUDA(cudaSetDevice(cfg.device));
  if (!promos.empty()) poll_promotions(false);
  if (n_req == 0) return;
  // host-tier items of the call, each staged once
  std::unordered_map<uint32_t, uint32_t> staged;  // item -> ring slot
  for (uint64_t i = 0; i < (uint64_t)n_req * k; ++i)
    for (uint32_t kind = 0; kind < 2; ++kind) {
      const uint32_t item = 2 * ids[i] + kind;
      if (loc[item].hbm_off == FreeList::kNone && !staged.count(item)) staged.emplace(item, (uint32_t)staged.size());
    }
  if (!staged.empty()) {
    ensure_ring();
    require(staged.size() <= slots, HR_ESTATE,
            "hr_attend: " + std::to_string(staged.size()) + " host-tier items exceed the staging ring (" +
                std::to_string(slots) + " slots); split the batch");
  }
  const uint64_t ns = (uint64_t)nl * lay.Hl;  // slabs of the window
  std::vector<uint8_t*> slot_codes(staged.size());
  std::vector<std::pair<uint32_t, uint32_t>> order_st(staged.begin(), staged.end());
  std::sort(order_st.begin(), order_st.end(), [](auto& x, auto& y) { return x.second < y.second; });
  for (const auto& [item, si] : order_st) {
    Slot& sl = ring[si];
    const uint32_t sc = scheme[item];
    const uint64_t cb = lay.code_bytes_slab(sc), ms = lay.meta_stride(sc);
    const uint64_t c0 = (uint64_t)l0 * lay.Hl * cb, cn = ns * cb;
    const uint64_t mo = lay.meta_offset(sc), m0 = mo + (uint64_t)l0 * lay.Hl * ms, mn = ns * ms;
    const uint64_t dst_m = align_up(cn, 256);  // window meta right after the window codes
    HR_CUDA(cudaStreamWaitEvent(copy_stream, sl.free_ev, 0));
    const uint8_t* src = loc[item].pin_off != FreeList::kNone    ? pin_base + loc[item].pin_off
                         : loc[item].page_off != FreeList::kNone ? page_base + loc[item].page_off
                         : loc[item].backing_off != FreeList::kNone ? backing_base + loc[item].backing_off
                                                                    : nullptr;
    const bool pinned_src = loc[item].pin_off != FreeList::kNone ||
                            (loc[item].page_off == FreeList::kNone && loc[item].backing_off != FreeList::kNone &&
                             backing_is_pinned);
    if (!pinned_src) {  // pageable or disk: the window through this slot's pinned bounce buffer
      ensure_bounce(sl);
      if (sl.used) HR_CUDA(cudaEventSynchronize(sl.copied));
      if (src) {
        host_copy(sl.bounce, src + c0, cn);
        if (mn) host_copy(sl.bounce + dst_m, src + m0, mn);
      } else {  // DISK tier: the blob, then the window out of it
        read_disk(item, sl.bounce);
        if (c0) std::memmove(sl.bounce, sl.bounce + c0, cn);
        if (mn) std::memmove(sl.bounce + dst_m, sl.bounce + m0, mn);
      }
      src = sl.bounce;
      HR_CUDA(cudaMemcpyAsync(sl.dev, src, dst_m + mn, cudaMemcpyHostToDevice, copy_stream));
    } else {
      HR_CUDA(cudaMemcpyAsync(sl.dev, src + c0, cn, cudaMemcpyHostToDevice, copy_stream));
      if (mn) HR_CUDA(cudaMemcpyAsync(sl.dev + dst_m, src + m0, mn, cudaMemcpyHostToDevice, copy_stream));
    }
    HR_CUDA(cudaEventRecord(sl.copied, copy_stream));
    sl.used = true;
    // the kernel addresses slab (l0 + l) * Hl + h from the descriptor: offset the pointers by the window start
    slot_codes[si] = sl.dev;
    stats.bytes_h2d += dst_m + mn;
    stats.h2d_items++;
  }
  const size_t n_desc = 2ull * n_req * k;
  DescBuf& db = desc_buffer(n_desc);
  for (uint32_t r = 0; r < n_req; ++r) {
    const bool counted = ((req_counter + r) % (uint64_t)cfg.world) == (uint64_t)cfg.rank;
    for (uint32_t j = 0; j < k; ++j)
      for (uint32_t kind = 0; kind < 2; ++kind) {
        const uint32_t item = 2 * ids[(uint64_t)r * k + j] + kind;
        const uint32_t sc = scheme[item];
        AsmDesc d{};
        const auto it = staged.find(item);
        if (it == staged.end()) {
          d.codes = hbm_ptr(item);
          d.meta = d.codes + lay.meta_offset(sc);
          stats.hits[HR_T_HBM]++;
        } else {
          const uint64_t cb = lay.code_bytes_slab(sc), ms = lay.meta_stride(sc);
          uint8_t* base = slot_codes[it->second];
          d.codes = base - (uint64_t)l0 * lay.Hl * cb;
          d.meta = base + align_up(ns * cb, 256) - (uint64_t)l0 * lay.Hl * ms;
          const Loc& l = loc[item];
          stats.hits[l.pin_off != FreeList::kNone ||
                             (l.page_off == FreeList::kNone && l.backing_off != FreeList::kNone && backing_is_pinned)
                         ? HR_T_PIN
                         : HR_T_PAGE]++;
        }
        d.count = counted ? reinterpret_cast<unsigned long long*>(delta + item) : nullptr;
        d.slot = j;
        d.scheme = sc;
        db.host[((uint64_t)r * k + j) * 2 + kind] = d;
        stats.bytes_hbm_alg += bytes_read_alg(item) / lay.L * nl;
      }
  }
  HR_CUDA(cudaMemcpyAsync(db.dev, db.host, n_desc * sizeof(AsmDesc), cudaMemcpyHostToDevice, st));
  for (const auto& kv : staged) HR_CUDA(cudaStreamWaitEvent(st, ring[kv.second].copied, 0));
  AttnParams p{};
  p.descs = db.dev;
  p.q = static_cast<const uint16_t*>(q);
  p.o = static_cast<uint16_t*>(o);
  p.lse = lse;
  p.kv_dump = static_cast<uint16_t*>(kv_dump);
  p.n_req = n_req, p.k = k, p.L = nl, p.l0 = l0, p.Hl = lay.Hl, p.T = lay.T, p.D = lay.D, p.g = g, p.n_q = n_q;
  p.own_k = static_cast<const uint16_t*>(k_own);
  p.own_v = static_cast<const uint16_t*>(v_own);
  p.n_own = k_own ? n_q : 0;
  p.M = g * n_q;
  p.G = lay.G, p.g_shift = (uint32_t)__builtin_ctz(lay.G), p.gse_e = lay.gse_e, p.gse_m = lay.gse_m;
  p.dtype = lay.dtype;
  const float sc = scale > 0.f ? scale : 1.f / std::sqrt((float)lay.D);
  p.scale_log2 = sc * 1.4426950408889634f;
  for (uint32_t s = 0; s < HR_N_SCHEMES; ++s) {
    p.code_slab[s] = lay.code_bytes_slab(s);
    p.meta_stride[s] = (uint32_t)lay.meta_stride(s);
  }
  // key splits when the call's units alone leave SMs idle (a per-layer prefill call: n_req * Hl units)
  if (!n_sms) HR_CUDA(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, cfg.device));
  const uint64_t units = (uint64_t)n_req * nl * lay.Hl;
  const char* fs = std::getenv("HARAG_ATT_SPLIT");  // tests / tuning: force the split count
  const uint32_t unit_tiles = k * (lay.T / 64) + (k_own ? 1u : 0u);
  p.n_split = fs ? (uint32_t)std::max(1, std::atoi(fs)) : attend_splits(units, unit_tiles, n_sms);
  p.n_split = std::min<uint32_t>(p.n_split, unit_tiles);
  if (p.n_split > 1) {
    const uint64_t need = units * p.n_split * 128ull * (lay.D + 1);
    // grown rarely: cudaFree waits for the launches still reading the old buffers
    if (need > att_part_floats) {
      if (att_part) HR_CUDA(cudaFree(att_part));
      att_part = nullptr;
      HR_CUDA(cudaMalloc((void**)&att_part, need * sizeof(float)));
      att_part_floats = need;
    }
    if (units > att_cnt_n) {
      if (att_cnt) HR_CUDA(cudaFree(att_cnt));
      att_cnt = nullptr;
      HR_CUDA(cudaMalloc((void**)&att_cnt, units * sizeof(uint32_t)));
      HR_CUDA(cudaMemset(att_cnt, 0, units * sizeof(uint32_t)));
      att_cnt_n = units;
    }
    p.part_o = att_part;
    p.part_lse = att_part + units * p.n_split * 128ull * lay.D;
    p.part_cnt = att_cnt;
    // the workspace is shared by every split launch of the store: order this one after the previous one
    // even when the caller alternates streams (a no-op wait on the same stream)
    if (att_done) HR_CUDA(cudaStreamWaitEvent(st, att_done, 0));
  }
  // q read + o written (algorithmic), beside the codes + meta counted above
  stats.bytes_hbm_alg += 2ull * 2 * n_req * nl * lay.Hl * g * n_q * lay.D;
  if (k_own) stats.bytes_hbm_alg += 2ull * 2 * n_req * nl * lay.Hl * n_q * lay.D;  // own K, V read
  cudaEvent_t a = nullptr, b = nullptr;
  if (timing) {
    HR_CUDA(cudaEventCreate(&a));
    HR_CUDA(cudaEventCreate(&b));
    HR_CUDA(cudaEventRecord(a, st));
  }
  launch_attend(p, st);
  if (p.n_split > 1) {
    if (!att_done) HR_CUDA(cudaEventCreateWithFlags(&att_done, cudaEventDisableTiming));
    HR_CUDA(cudaEventRecord(att_done, st));
  }
  if (timing) {
    HR_CUDA(cudaEventRecord(b, st));
    timers.emplace_back(a, b);
  }
  stats.kernel_launches++;
  for (const auto& kv : staged) HR_CUDA(cudaEventRecord(ring[kv.second].free_ev, st));
  HR_CUDA(cudaEventRecord(db.done, st));
  req_counter += n_req;
  stats.requests += n_req;
}

void Store::replace(cudaStream_t st) {
  require(state == State::Built, HR_ESTATE, "hr_replace before the store is built");
  const NvtxRange nvtx_call("hr_replace");
  const CpuBind bind(local_cpus);  // pinned-tier fills
  HR_CUDA(cudaSetDevice(cfg.device));
  std::vector<int64_t> dh(n_items);
  HR_CUDA(cudaMemcpyAsync(dh.data(), delta, sizeof(int64_t) * n_items, cudaMemcpyDeviceToHost, st));
  HR_CUDA(cudaStreamSynchronize(st));
  // the epoch is computed on copies and committed only once it is known to be applicable, so a
  // refused re-placement (HR_ESTATE) leaves hotness, rank order and delta untouched
  std::vector<uint64_t> h_new(h);
  epoch_update(h_new.data(), dh.data(), n_items, cfg.decay_shift);  // a9 (R20)
  std::vector<uint32_t> order_new = rank_items(h_new.data(), n_items);
  std::swap(order, order_new);
  std::vector<uint32_t> nt = place_lists();  // Alg. 2 step 1 over the new order
  std::swap(order, order_new);
  if (!alg2) {
    if (cfg.backing_pinned && !on_disk)
      for (auto& t : nt)
        if (t == HR_T_PAGE) t = HR_T_PIN;
    poll_promotions(true);  // the previous epoch's copies (normally long done)
    bool any_move = false;
    for (uint32_t i = 0; i < n_items; ++i) any_move |= (nt[i] == HR_T_HBM) != (loc[i].hbm_off != FreeList::kNone);
    require(!any_move || cfg.keep_backing || disk_fd >= 0, HR_ESTATE, "re-placement needs keep_backing = 1");
  }
  h.swap(h_new);
  order.swap(order_new);
  HR_CUDA(cudaMemsetAsync(delta, 0, sizeof(int64_t) * n_items, st));
  if (alg2) {  // demand mode (R20): only the lists change; stale queue entries leave by LRU
    alg2->set_lists(nt.data());
    return;
  }
  if (!mig_ev) HR_CUDA(cudaEventCreateWithFlags(&mig_ev, cudaEventDisableTiming));
  HR_CUDA(cudaEventRecord(mig_ev, st));
  HR_CUDA(cudaStreamWaitEvent(copy_stream, mig_ev, 0));
  bool pin_changed = false;
  // evict first (host copies are inclusive, R16)
  for (uint32_t i = 0; i < n_items; ++i) {
    if (nt[i] != HR_T_HBM && loc[i].hbm_off != FreeList::kNone) {
      hbm.release(loc[i].hbm_off, bytes[i]);
      loc[i].hbm_off = FreeList::kNone;
      stats.migrations_out++;
    }
    if (nt[i] != HR_T_PIN && loc[i].pin_off != FreeList::kNone) {
      pin.release(loc[i].pin_off, bytes[i]);
      loc[i].pin_off = FreeList::kNone;
      pin_changed = true;
    }
    if (nt[i] != HR_T_PAGE && loc[i].page_off != FreeList::kNone) {
      page.release(loc[i].page_off, bytes[i]);
      loc[i].page_off = FreeList::kNone;
    }
  }
  // pinned space freed above may still be the source of an in-flight DMA
  if (pin_changed) HR_CUDA(cudaStreamSynchronize(copy_stream));
  // promote in rank order
  for (uint32_t pos = 0; pos < n_items; ++pos) {
    const uint32_t i = order[pos];
    if (nt[i] == HR_T_HBM && loc[i].hbm_off == FreeList::kNone) {
      uint64_t off = hbm.alloc(bytes[i]);
      if (off == FreeList::kNone && hbm_cap - hbm.used() >= align_up(bytes[i], FreeList::kAlign)) {
        // the lists fit the budget by construction: defragment (needs an idle device) and retry
        HR_CUDA(cudaDeviceSynchronize());
        poll_promotions(true);
        compact_hbm();
        off = hbm.alloc(bytes[i]);
      }
      if (off == FreeList::kNone) {
        stats.failed_promotions++;
        nt[i] = on_disk ? HR_T_DISK : cfg.backing_pinned ? HR_T_PIN : HR_T_PAGE;
        continue;
      }
      if (loc[i].backing_off != FreeList::kNone && backing_is_pinned) {
        HR_CUDA(cudaMemcpyAsync(hbm_base + off, backing_base + loc[i].backing_off, bytes[i], cudaMemcpyHostToDevice,
                                copy_stream));
      } else if (loc[i].backing_off != FreeList::kNone) {
        // pageable backing: through the staging ring's pinned bounce buffers, round robin, so the
        // host copy of one promotion overlaps the DMA of the previous ones (a cudaMemcpyAsync straight
        // from pageable memory is staged by the driver at ~11 GB/s and blocks the host)
        ensure_ring();
        Slot& sl = ring[promo_slot++ % slots];
        ensure_bounce(sl);
        if (sl.used) HR_CUDA(cudaEventSynchronize(sl.copied));  // the bounce's previous DMA is done
        host_copy(sl.bounce, backing_base + loc[i].backing_off, bytes[i]);
        HR_CUDA(cudaMemcpyAsync(hbm_base + off, sl.bounce, bytes[i], cudaMemcpyHostToDevice, copy_stream));
        HR_CUDA(cudaEventRecord(sl.copied, copy_stream));
        sl.used = true;
      } else {  // disk-backed: through a pinned bounce, one item at a time
        ensure_ring();
        Slot& sl = ring[0];
        ensure_bounce(sl);
        HR_CUDA(cudaStreamSynchronize(copy_stream));
        read_disk(i, sl.bounce);
        HR_CUDA(cudaMemcpyAsync(hbm_base + off, sl.bounce, bytes[i], cudaMemcpyHostToDevice, copy_stream));
        // the next user of this bounce buffer (a streamed item of hr_assemble_kv) waits for the DMA
        HR_CUDA(cudaEventRecord(sl.copied, copy_stream));
        sl.used = true;
      }
      Promo pr{i, off, nullptr};
      HR_CUDA(cudaEventCreateWithFlags(&pr.ev, cudaEventDisableTiming));
      HR_CUDA(cudaEventRecord(pr.ev, copy_stream));
      promos.push_back(pr);
      stats.migrations_in++;
      stats.bytes_migrated += bytes[i];
    } else if (nt[i] == HR_T_PAGE && page_base && loc[i].page_off == FreeList::kNone) {
      const uint64_t off = page.alloc(bytes[i]);  // (no compaction: a miss falls back to DISK)
      if (off == FreeList::kNone) {
        nt[i] = HR_T_DISK;
        continue;
      }
      loc[i].page_off = off;
      fill_host(i, page_base + off);
    } else if (nt[i] == HR_T_PIN && pin_base && loc[i].pin_off == FreeList::kNone) {
      uint64_t off = pin.alloc(bytes[i]);
      if (off == FreeList::kNone && pin_cap - pin.used() >= align_up(bytes[i], FreeList::kAlign)) {
        HR_CUDA(cudaStreamSynchronize(copy_stream));
        compact_pin();
        off = pin.alloc(bytes[i]);
      }
      if (off == FreeList::kNone) {
        nt[i] = on_disk ? HR_T_DISK : HR_T_PAGE;
        continue;
      }
      loc[i].pin_off = off;
      fill_host(i, pin_base + off);
    }
  }
  tier = nt;  // target placement; HBM promotions become resident as their copies land
}

void Store::compact_hbm() {
  std::vector<std::pair<uint64_t, uint32_t>> res;
  for (uint32_t i = 0; i < n_items; ++i)
    if (loc[i].hbm_off != FreeList::kNone) res.emplace_back(loc[i].hbm_off, i);
  std::sort(res.begin(), res.end());
  uint8_t* tmp = nullptr;
  uint64_t cursor = 0;
  for (auto& r : res) {
    const uint32_t i = r.second;
    const uint64_t sz = align_up(bytes[i], FreeList::kAlign);
    if (r.first != cursor) {
      if (r.first - cursor >= sz) {
        HR_CUDA(cudaMemcpyAsync(hbm_base + cursor, hbm_base + r.first, bytes[i], cudaMemcpyDeviceToDevice,
                                copy_stream));
      } else {  // overlapping move: through a bounce buffer
        if (!tmp) HR_CUDA(cudaMalloc(&tmp, max_item));
        HR_CUDA(cudaMemcpyAsync(tmp, hbm_base + r.first, bytes[i], cudaMemcpyDeviceToDevice, copy_stream));
        HR_CUDA(cudaMemcpyAsync(hbm_base + cursor, tmp, bytes[i], cudaMemcpyDeviceToDevice, copy_stream));
      }
      loc[i].hbm_off = cursor;
    }
    cursor += sz;
  }
  HR_CUDA(cudaStreamSynchronize(copy_stream));
  if (tmp) HR_CUDA(cudaFree(tmp));
  hbm.reset_compacted(cursor, hbm_cap);
  compactions++;
}

void Store::compact_pin() {  // host-side twin of compact_hbm (no DMA reads the pinned tier here)
  std::vector<std::pair<uint64_t, uint32_t>> res;
  for (uint32_t i = 0; i < n_items; ++i)
    if (loc[i].pin_off != FreeList::kNone) res.emplace_back(loc[i].pin_off, i);
  std::sort(res.begin(), res.end());
  uint64_t cursor = 0;
  for (auto& r : res) {
    const uint32_t i = r.second;
    if (r.first != cursor) {
      std::memmove(pin_base + cursor, pin_base + r.first, bytes[i]);
      loc[i].pin_off = cursor;
    }
    cursor += align_up(bytes[i], FreeList::kAlign);
  }
  pin.reset_compacted(cursor, pin_cap);
}

// ------------------------------------------------------------ persistence
namespace {
constexpr char kMagic[8] = {'H', 'R', 'S', 'T', 'O', 'R', 'E', '1'};
struct FileHeader {
  char magic[8];
  uint32_t version, n_docs;
  uint64_t data_offset;
  hr_store_config cfg;
};
std::string errno_msg(const char* what, const std::string& path) { return std::string(what) + " " + path + ": " + std::strerror(errno); }
void pwrite_all(int fd, const void* buf, size_t n, uint64_t off, const std::string& path) {
  const uint8_t* p = (const uint8_t*)buf;
  while (n) {
    const ssize_t w = ::pwrite(fd, p, n, (off_t)off);
    require(w > 0, HR_EINVAL, errno_msg("write", path));
    p += w, n -= (size_t)w, off += (uint64_t)w;
  }
}
void pread_all(int fd, void* buf, size_t n, uint64_t off, const std::string& path) {
  uint8_t* p = (uint8_t*)buf;
  while (n) {
    const ssize_t r = ::pread(fd, p, n, (off_t)off);
    require(r > 0, HR_EINVAL, errno_msg("read", path));
    p += r, n -= (size_t)r, off += (uint64_t)r;
  }
}
}  // namespace

std::vector<uint64_t> Store::file_offsets(uint64_t data_offset) const {
  std::vector<uint64_t> off(n_items);
  uint64_t o = data_offset;
  for (uint32_t i = 0; i < n_items; ++i) off[i] = o, o += align_up(bytes[i], 4096);
  return off;
}

void Store::save(const char* path) const {
  require(state == State::Built, HR_ESTATE, "hr_store_save before the store is built");
  const std::string P(path);
  const int fd = ::open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
  require(fd >= 0, HR_EINVAL, errno_msg("open", P));
  FileHeader hd{};
  std::memcpy(hd.magic, kMagic, 8);
  hd.version = 1;
  hd.n_docs = n_docs;
  hd.cfg = cfg;
  const uint64_t arrays = sizeof(FileHeader) + n_items * (sizeof(uint64_t) + sizeof(uint32_t));
  hd.data_offset = align_up(arrays, 4096);
  std::vector<uint8_t> head(hd.data_offset, 0);
  std::memcpy(head.data(), &hd, sizeof hd);
  std::memcpy(head.data() + sizeof hd, h.data(), n_items * sizeof(uint64_t));
  std::memcpy(head.data() + sizeof hd + n_items * sizeof(uint64_t), scheme.data(), n_items * sizeof(uint32_t));
  try {
    pwrite_all(fd, head.data(), head.size(), 0, P);
    const std::vector<uint64_t> off = file_offsets(hd.data_offset);
    std::vector<uint8_t> buf(align_up(max_item, 4096));
    for (uint32_t i = 0; i < n_items; ++i) {
      std::memset(buf.data() + bytes[i], 0, buf.size() - bytes[i]);
      size_t len = 0;
      export_item(i, buf.data(), buf.size(), &len);
      pwrite_all(fd, buf.data(), align_up(bytes[i], 4096), off[i], P);
    }
  } catch (...) {
    ::close(fd);
    throw;
  }
  require(::close(fd) == 0, HR_EINVAL, errno_msg("close", P));
}

void Store::build_from_file(const char* path, cudaStream_t st) {
  require(state == State::Empty, HR_ESTATE, "store already built");
  const CpuBind bind(local_cpus);
  const std::string P(path);
  const int fd = ::open(path, O_RDONLY);
  require(fd >= 0, HR_EINVAL, errno_msg("open", P));
  disk_fd = fd;  // owned by the store from here on
  disk_path = P;
  FileHeader hd{};
  pread_all(fd, &hd, sizeof hd, 0, P);
  require(std::memcmp(hd.magic, kMagic, 8) == 0 && hd.version == 1, HR_ECORRUPT, P + " is not a harag store file");
  const hr_store_config& f = hd.cfg;
  require(f.L == cfg.L && f.H == cfg.H && f.D == cfg.D && f.T == cfg.T && f.dtype == cfg.dtype &&
              (f.group ? f.group : f.D) == (cfg.group ? cfg.group : cfg.D) && f.gse_ebits == cfg.gse_ebits &&
              f.gse_mbits == cfg.gse_mbits && f.rank == cfg.rank && f.world == cfg.world,
          HR_EINVAL, "store file shape differs from the store config");
  const uint32_t nd = hd.n_docs, ni = 2 * nd;
  std::vector<uint64_t> hot(ni);
  std::vector<uint32_t> sc(ni);
  pread_all(fd, hot.data(), ni * sizeof(uint64_t), sizeof hd, P);
  pread_all(fd, sc.data(), ni * sizeof(uint32_t), sizeof hd + ni * sizeof(uint64_t), P);
  for (uint32_t v : sc) require(v < HR_N_SCHEMES, HR_ECORRUPT, "bad scheme in store file");
  const bool on_disk = cfg.disk_backing != 0;
  setup(nd, hot.data(), std::move(sc), on_disk);
  disk_off = file_offsets(hd.data_offset);
  if (on_disk) {  // cold reads bypass the page cache when the filesystem allows it
    disk_fd_direct = ::open(path, O_RDONLY | O_DIRECT);
    if (disk_fd_direct < 0) disk_fd_direct = -1;
  }
  ensure_ring();
  Slot& sl = ring[0];
  ensure_bounce(sl);
  for (uint32_t i = 0; i < n_items; ++i) {
    const uint64_t rb = align_up(bytes[i], 4096);
    if (loc[i].hbm_off != FreeList::kNone) {  // GPU_LIST: file -> pinned bounce -> HBM arena
      HR_CUDA(cudaStreamSynchronize(st));
      read_disk(i, sl.bounce);
      HR_CUDA(cudaMemcpyAsync(hbm_ptr(i), sl.bounce, bytes[i], cudaMemcpyHostToDevice, st));
    }
    if (loc[i].pin_off != FreeList::kNone) pread_all(fd, pin_base + loc[i].pin_off, bytes[i], disk_off[i], P);
    if (loc[i].page_off != FreeList::kNone) pread_all(fd, page_base + loc[i].page_off, bytes[i], disk_off[i], P);
    if (loc[i].backing_off != FreeList::kNone && !backing_filled.count(loc[i].backing_off)) {
      pread_all(fd, backing_base + loc[i].backing_off, rb > bytes[i] ? bytes[i] : rb, disk_off[i], P);
      backing_filled.insert(loc[i].backing_off);
    }
  }
  HR_CUDA(cudaStreamSynchronize(st));
  n_put = n_docs;
  cudaFree(scratch);
  scratch = nullptr;
  scratch_items = 0;
  state = State::Built;
}

// One item's blob from the store file into a page-aligned host buffer (>= align4096(bytes)):
// O_DIRECT reads of 4 MiB pieces spread over the worker pool.
void Store::read_disk(uint32_t item, uint8_t* dst) {
  const int fd = disk_fd_direct >= 0 ? disk_fd_direct : disk_fd;
  require(fd >= 0, HR_ESTATE, "item has no host copy");
  const uint64_t n = align_up(bytes[item], 4096), off = disk_off[item];
  constexpr uint64_t kPiece = 4u << 20;
  const unsigned pieces = (unsigned)((n + kPiece - 1) / kPiece);
  if (!copy_pool) host_copy(nullptr, nullptr, 0);  // creates the pool
  std::atomic<int> err{0};
  for (unsigned b = 0; b < pieces; b += copy_pool->size()) {
    copy_pool->parallel_for(std::min(copy_pool->size(), pieces - b), [&](unsigned p) {
      const uint64_t o = (uint64_t)(b + p) * kPiece;
      const uint64_t len = std::min(kPiece, n - o);
      uint8_t* d = dst + o;
      uint64_t done = 0;
      while (done < len) {
        const ssize_t r = ::pread(fd, d + done, len - done, (off_t)(off + o + done));
        if (r <= 0) {
          err = errno ? errno : EIO;
          return;
        }
        done += (uint64_t)r;
      }
    });
  }
  require(err == 0, HR_EINVAL, "read " + disk_path + ": " + std::strerror(err));
}

void Store::export_item(uint32_t item, void* dst, size_t cap, size_t* len) const {
  require(state == State::Built, HR_ESTATE, "store not built");
  require(item < n_items, HR_ENOTFOUND, "item id out of range");
  if (len) *len = bytes[item];
  require(cap >= bytes[item], HR_EINVAL, "destination too small");
  if (loc[item].hbm_off != FreeList::kNone) {
    HR_CUDA(cudaSetDevice(cfg.device));
    HR_CUDA(cudaDeviceSynchronize());
    HR_CUDA(cudaMemcpy(dst, hbm_ptr(item), bytes[item], cudaMemcpyDeviceToHost));
  } else if (loc[item].pin_off != FreeList::kNone) {
    std::memcpy(dst, pin_base + loc[item].pin_off, bytes[item]);
  } else if (loc[item].page_off != FreeList::kNone) {
    std::memcpy(dst, page_base + loc[item].page_off, bytes[item]);
  } else if (loc[item].backing_off != FreeList::kNone) {
    std::memcpy(dst, backing_base + loc[item].backing_off, bytes[item]);
  } else {
    require(disk_fd >= 0 && !disk_off.empty(), HR_ESTATE, "item has no copy");
    pread_all(disk_fd, dst, bytes[item], disk_off[item], disk_path);
  }
}

uint64_t Store::placement_hash() const {
  require(state == State::Built, HR_ESTATE, "store not built");
  uint64_t x = 0xcbf29ce484222325ull;  // FNV-1a, 64-bit
  auto mix = [&x](uint64_t v) {
    for (int b = 0; b < 8; ++b) x = (x ^ ((v >> (8 * b)) & 0xFF)) * 0x100000001b3ull;
  };
  mix(n_items);
  for (uint32_t i = 0; i < n_items; ++i) {
    mix(h[i]);
    mix(scheme[i]);
    mix(logical_tier(i));
  }
  for (uint32_t i = 0; i < n_items; ++i) mix(order[i]);
  return x;
}

void Store::get_stats(hr_stats* out) {
  // HARAG_TIMELINE=<file>: append the timed launches and host-tier copy windows (start, duration in ms,
  // relative to the first timed launch) — a poor man's timeline where no Nsight Systems is available
  if (const char* tl = std::getenv("HARAG_TIMELINE"); tl && !timers.empty()) {
    if (FILE* f = std::fopen(tl, "a")) {
      cudaEvent_t ref = timers.front().first;
      HR_CUDA(cudaEventSynchronize(timers.back().second));
      for (auto& t : timers) {
        float a = 0, d = 0;
        cudaEventElapsedTime(&a, ref, t.first);
        cudaEventElapsedTime(&d, t.first, t.second);
        std::fprintf(f, "kernel %.4f %.4f\n", a, d);
      }
      for (auto& t : h2d_timers) {
        float a = 0, d = 0;
        cudaEventSynchronize(t.second);
        cudaEventElapsedTime(&a, ref, t.first);
        cudaEventElapsedTime(&d, t.first, t.second);
        std::fprintf(f, "h2d %.4f %.4f\n", a, d);
      }
      std::fclose(f);
    }
  }
  if (!timers.empty()) {
    for (auto& t : timers) {
      HR_CUDA(cudaEventSynchronize(t.second));
      float ms = 0;
      HR_CUDA(cudaEventElapsedTime(&ms, t.first, t.second));
      stats.kernel_ms += ms;
      stats.timed_launches++;
      cudaEventDestroy(t.first);
      cudaEventDestroy(t.second);
    }
    timers.clear();
  }
  for (auto& t : qtimers) {
    HR_CUDA(cudaEventSynchronize(t.second));
    float ms = 0;
    HR_CUDA(cudaEventElapsedTime(&ms, t.first, t.second));
    stats.quant_ms += ms;
    stats.quant_launches++;
    cudaEventDestroy(t.first);
    cudaEventDestroy(t.second);
  }
  qtimers.clear();
  for (auto& t : h2d_timers) {
    HR_CUDA(cudaEventSynchronize(t.second));
    float ms = 0;
    HR_CUDA(cudaEventElapsedTime(&ms, t.first, t.second));
    stats.h2d_ms += ms;
    cudaEventDestroy(t.first);
    cudaEventDestroy(t.second);
  }
  h2d_timers.clear();
  stats.hbm_used = hbm.used();
  stats.pin_used = pin.used();
  *out = stats;
}

}  // namespace harag
