// The HA-RAG store (one per rank / GPU).  See store.cpp and DESIGN.md §1, §4.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdint>
#include <map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "layout.h"
#include "numa.h"
#include "pool.h"
#include "policy.h"

#include <memory>
#include <string>

namespace harag {

// First-fit free list over one contiguous region (HBM arena / pinned tier).
class FreeList {
 public:
  static constexpr uint64_t kAlign = 256;
  static constexpr uint64_t kNone = ~0ull;
  void reset(uint64_t cap) {
    free_.clear();
    used_ = 0;
    if (cap) free_[0] = cap;
  }
  uint64_t alloc(uint64_t size);  // kNone when no contiguous block fits
  void release(uint64_t off, uint64_t size);
  uint64_t used() const { return used_; }
  // after compaction: [0, end) in use, [end, cap) one free block
  void reset_compacted(uint64_t end, uint64_t cap) {
    free_.clear();
    if (cap > end) free_[end] = cap - end;
    used_ = end;
  }

 private:
  std::map<uint64_t, uint64_t> free_;  // offset -> size
  uint64_t used_ = 0;
};

struct Store {
  enum class State { Empty, Building, Built };
  struct Loc {
    uint64_t hbm_off = FreeList::kNone;      // HBM arena copy
    uint64_t pin_off = FreeList::kNone;      // pinned-tier copy
    uint64_t backing_off = FreeList::kNone;  // host backing copy
    uint64_t page_off = FreeList::kNone;     // pageable PAGE-tier cache copy (disk-backed stores)
    bool backing_alias = false;
  };
  struct DescBuf {
    AsmDesc* dev = nullptr;
    AsmDesc* host = nullptr;  // pinned
    size_t cap = 0;
    cudaEvent_t done = nullptr;
  };
  struct Slot {  // host-tier staging ring slot
    uint8_t* dev = nullptr;
    uint8_t* bounce = nullptr;  // pinned bounce buffer for pageable items
    cudaEvent_t copied = nullptr, free_ev = nullptr;
    bool used = false;
  };
  static constexpr int kDescBufs = 8;

  explicit Store(const hr_store_config& c);
  ~Store();

  void build_begin(uint32_t n_docs, const uint64_t* hotness, const uint32_t* schemes = nullptr);
  void setup(uint32_t n_docs, const uint64_t* hotness, std::vector<uint32_t> schemes, bool disk);
  std::vector<uint32_t> place_lists() const;  // Alg. 2 step 1 by bytes for this store's tiers
  void save(const char* path) const;
  void build_from_file(const char* path, cudaStream_t st);
  void read_disk(uint32_t item, uint8_t* dst);
  std::vector<uint64_t> file_offsets(uint64_t data_offset) const;
  void build_put(uint32_t doc, const void* k_src, const void* v_src, cudaStream_t st);
  void build_put_batch(uint32_t n, const uint32_t* docs, const void* const* k_srcs, const void* const* v_srcs,
                       cudaStream_t st);
  void build_end(cudaStream_t st);
  void build_with_source(uint32_t n_docs, const uint64_t* hotness, hr_src_fn src, void* user, cudaStream_t st);
  void assemble(uint32_t n_req, uint32_t k, const uint32_t* ids, void* const* k_out, void* const* v_out,
                cudaStream_t st);
  void replace(cudaStream_t st);
  void attend(uint32_t n_req, uint32_t k, const uint32_t* ids, uint32_t l0, uint32_t nl, const void* q, uint32_t n_q,
              uint32_t g, void* o, float* lse, float scale, void* kv_dump, cudaStream_t st,
              const void* k_own = nullptr, const void* v_own = nullptr);
  void export_item(uint32_t item, void* dst, size_t cap, size_t* len) const;
  void get_stats(hr_stats* out);

  uint8_t* hbm_ptr(uint32_t item) const;
  uint64_t backing_key(uint32_t item) const;
  uint64_t bytes_read_alg(uint32_t item) const;
  DescBuf& desc_buffer(size_t n);
  void ensure_ring();
  void ensure_bounce(Slot& sl);            // pinned bounce buffers of every slot, placement-probed
  std::vector<uint8_t*> bounce_rejects;    // slow-probing pinned buffers, held until close
  double bounce_best_gbps = 0;
  void launch(const AsmDesc* dev_descs, const AsmDesc* host_descs, uint32_t n, uint32_t k, uint32_t scheme_mask,
              cudaStream_t st);
  void compact_hbm();
  void validate_request(uint32_t n_req, uint32_t k, const uint32_t* ids, void* const* k_out,
                        void* const* v_out) const;
  void release_deferred();
  void host_copy(void* dst, const void* src, size_t n);
  void fill_host(uint32_t item, uint8_t* dst);
  uint32_t logical_tier(uint32_t item) const;
  void compact_pin();

  uint64_t placement_hash() const;

  hr_store_config cfg;
  Layout lay;
  std::vector<int> local_cpus;  // numa_bind: CPUs local to the device (empty: unbound)
  State state = State::Empty;
  uint32_t n_docs = 0, n_items = 0, n_put = 0;
  uint32_t slots = 3;
  std::vector<uint64_t> h;       // hotness per item (AF)
  std::vector<uint32_t> scheme;  // Alg. 1 result
  std::vector<uint64_t> bytes;   // packed blob bytes per item
  std::vector<uint32_t> order;   // hotness rank order
  std::vector<uint32_t> tier;    // current tier per item
  std::vector<Loc> loc;
  std::vector<uint8_t> put_done;
  std::unordered_set<uint64_t> backing_filled;
  uint64_t max_item = 0;

  uint8_t* hbm_base = nullptr;
  uint64_t hbm_cap = 0;
  FreeList hbm;
  uint64_t compactions = 0;
  uint8_t* pin_base = nullptr;
  uint64_t pin_cap = 0;
  FreeList pin;
  uint8_t* page_base = nullptr;  // PAGE tier cache of a disk-backed store (pageable)
  uint64_t page_cap = 0;
  FreeList page;
  bool on_disk = false;
  uint8_t* backing_base = nullptr;
  uint64_t backing_bytes = 0;
  bool backing_is_pinned = false;

  int64_t* delta = nullptr;  // device int64[n_items] hotness delta (a1)
  int* err_flag = nullptr;
  uint8_t* scratch = nullptr;  // build: quantised blobs headed for the host
  uint32_t scratch_items = 0;  // capacity of scratch in items of max_item bytes
  static constexpr uint32_t kPutBatch = 16;  // docs per hr_build_put_batch call (one quantize launch)
  static constexpr uint32_t kSrcBatch = 4;   // docs per launch in hr_build_store (source buffers: 4 x K+V)
  int* gse_range = nullptr;    // build: GSE-8 per-slab exponent range scratch
  void* src_k = nullptr;
  void* src_v = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::vector<DescBuf> dbuf;
  std::vector<AsmDesc> hdesc;  // host copy of an assemble call's descriptors
  int dbuf_next = 0;
  std::vector<Slot> ring;
  uint32_t promo_slot = 0;  // round-robin bounce slot of hr_replace's pageable promotions
  uint64_t req_counter = 0;
  // hr_attend key-split workspace (grown on demand): partial O / LSE and the per-unit arrival counters
  float* att_part = nullptr;
  uint64_t att_part_floats = 0;
  uint32_t* att_cnt = nullptr;
  uint64_t att_cnt_n = 0;
  cudaEvent_t att_done = nullptr;  // the last key-split launch: a split launch on another stream waits for it
  int n_sms = 0;
  // assemble tail balancing: per-launch claim counters (64 slots of 16 B, zero between launches)
  uint32_t* asm_sched = nullptr;
  uint32_t asm_sched_next = 0;
  uint32_t asm_dyn_pct = 25, asm_dyn_per_cta = 8;

  bool timing = false;       // CUDA events around every assemble launch (stats.kernel_ms)
  bool call_timing = false;  // CUDA events around every hr_assemble_kv call (hr_last_call_ms)
  bool call_recorded = false;
  cudaEvent_t call_ev[2] = {nullptr, nullptr};
  double last_call_ms();
  // HARAG_HOST_PROF=1: host-time breakdown of hr_assemble_kv, printed when the store is destroyed
  bool host_prof = false;
  // HARAG_METRICS_JSONL=<file>: one JSON line per hr_assemble_kv call (hits per tier, bytes, host time)
  FILE* metrics = nullptr;
  uint64_t metrics_calls = 0;
  double prof_ms[6] = {0, 0, 0, 0, 0, 0};
  uint64_t prof_calls = 0;
  std::chrono::steady_clock::time_point prof_t;
  int grid_override = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timers;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> h2d_timers;  // copy-stream window per assemble call
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> qtimers;     // quantize launches (hr_build_put*)
  std::unique_ptr<CopyPool> copy_pool;                           // pageable -> pinned bounce workers
  // demand mode (cfg.demand_mode = 1): the paper-literal Alg. 2 step 2 state machine
  std::unique_ptr<Alg2> alg2;
  std::vector<std::pair<uint64_t, uint64_t>> pending_pin_free, pending_page_free;  // (off, bytes)
  cudaEvent_t start_ev = nullptr;
  cudaEvent_t after_a_ev = nullptr;  // recorded after launch A when a promotion reuses space it reads
  // eager re-placement: asynchronous promotions (item becomes resident when its copy event completes)
  struct Promo {
    uint32_t item;
    uint64_t off;
    cudaEvent_t ev;
  };
  std::vector<Promo> promos;
  cudaEvent_t mig_ev = nullptr;
  // disk tier (hr_build_from_file): the store file backs items without a host copy
  int disk_fd = -1, disk_fd_direct = -1;
  std::string disk_path;
  std::vector<uint64_t> disk_off;
  void poll_promotions(bool wait_all);
  hr_stats stats{};
};

}  // namespace harag
