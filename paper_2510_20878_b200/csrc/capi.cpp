// extern "C" boundary of libharag (include/harag.h): argument marshalling and
// error translation only — every step runs in store.cpp / policy.cpp / the
// sm_100a kernels.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>

#include "analysis.h"
#include "harag.h"
#include "layout.h"
#include "policy.h"
#include "store.h"

struct hr_store {
  harag::Store impl;
  explicit hr_store(const hr_store_config& c) : impl(c) {}
};
struct hr_alg2 {
  harag::Alg2 impl;
  template <class... A>
  explicit hr_alg2(A&&... a) : impl(std::forward<A>(a)...) {}
};

namespace {
thread_local std::string g_err;

template <class F>
hr_status guard(F&& f) {
  try {
    f();
    return HR_OK;
  } catch (const harag::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return HR_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HR_EINVAL;
  }
}
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
#define NONNULL(p) harag::require((p) != nullptr, HR_EINVAL, #p " is NULL")
}  // namespace

extern "C" {

const char* hr_last_error(void) { return g_err.c_str(); }
uint32_t hr_abi_version(void) { return HR_ABI_VERSION; }

void hr_config_default(hr_store_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->L = 32, c->H = 8, c->D = 128, c->T = 512;  // Llama-3-8B KV shape, 512-token chunks
  c->dtype = HR_BF16;
  c->group = 0;
  c->gse_ebits = 4, c->gse_mbits = 3;  // 1+4+3
  c->n_ladder = 4;                     // INT8 -> E4M3 -> E5M2 -> GSE-8
  c->ladder[0] = HR_S_INT8, c->ladder[1] = HR_S_FP8E4M3, c->ladder[2] = HR_S_FP8E5M2, c->ladder[3] = HR_S_GSE8;
  c->tau[0] = c->tau[1] = c->tau[2] = 0.10;
  c->keep_backing = 1;
  c->decay_shift = 1;
  c->world = 1;
  c->staging_slots = 0;
  c->numa_bind = 1;
}

hr_status hr_store_create(const hr_store_config* cfg, hr_store** out) {
  return guard([&] {
    NONNULL(cfg);
    NONNULL(out);
    *out = nullptr;
    *out = new hr_store(*cfg);
  });
}

void hr_store_destroy(hr_store* s) { delete s; }

hr_status hr_build_store(hr_store* s, uint32_t n_docs, const uint64_t* hotness, hr_src_fn src, void* user,
                         void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.build_with_source(n_docs, hotness, src, user, S(stream));
  });
}
hr_status hr_build_begin(hr_store* s, uint32_t n_docs, const uint64_t* hotness) {
  return guard([&] {
    NONNULL(s);
    s->impl.build_begin(n_docs, hotness);
  });
}
hr_status hr_build_begin_schemes(hr_store* s, uint32_t n_docs, const uint64_t* hotness, const uint32_t* schemes) {
  return guard([&] {
    NONNULL(s);
    NONNULL(schemes);
    s->impl.build_begin(n_docs, hotness, schemes);
  });
}
hr_status hr_build_put(hr_store* s, uint32_t doc, const void* k_src, const void* v_src, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.build_put(doc, k_src, v_src, S(stream));
  });
}
hr_status hr_build_put_batch(hr_store* s, uint32_t n, const uint32_t* docs, const void* const* k_srcs,
                             const void* const* v_srcs, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.build_put_batch(n, docs, k_srcs, v_srcs, S(stream));
  });
}
hr_status hr_build_end(hr_store* s, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.build_end(S(stream));
  });
}

size_t hr_kv_bytes(const hr_store* s, uint32_t k) { return s ? s->impl.lay.kv_bytes(k) : 0; }

hr_status hr_assemble_kv(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, void* const* k_out,
                         void* const* v_out, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.assemble(n_req, k, doc_ids, k_out, v_out, S(stream));
  });
}

hr_status hr_hotness_delta(hr_store* s, int64_t** dev_ptr, uint32_t* n) {
  return guard([&] {
    NONNULL(s);
    NONNULL(dev_ptr);
    NONNULL(n);
    harag::require(s->impl.state == harag::Store::State::Built, HR_ESTATE, "store not built");
    *dev_ptr = s->impl.delta;
    *n = s->impl.n_items;
  });
}
hr_status hr_attend(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, const void* q_dev,
                    uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev, float scale, void* kv_dump,
                    void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.attend(n_req, k, doc_ids, 0, s->impl.lay.L, q_dev, n_q, g, o_dev, lse_dev, scale, kv_dump, S(stream));
  });
}
hr_status hr_attend_layers(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, uint32_t layer0,
                           uint32_t n_layers, const void* q_dev, uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev,
                           float scale, void* kv_dump, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.attend(n_req, k, doc_ids, layer0, n_layers, q_dev, n_q, g, o_dev, lse_dev, scale, kv_dump, S(stream));
  });
}
hr_status hr_attend_prefill(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, uint32_t layer0,
                            uint32_t n_layers, const void* q_dev, const void* k_own_dev, const void* v_own_dev,
                            uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev, float scale, void* stream) {
  return guard([&] {
    NONNULL(s);
    NONNULL(k_own_dev);
    NONNULL(v_own_dev);
    s->impl.attend(n_req, k, doc_ids, layer0, n_layers, q_dev, n_q, g, o_dev, lse_dev, scale, nullptr, S(stream),
                   k_own_dev, v_own_dev);
  });
}

hr_status hr_replace(hr_store* s, void* stream) {
  return guard([&] {
    NONNULL(s);
    s->impl.replace(S(stream));
  });
}

hr_status hr_store_save(const hr_store* s, const char* path) {
  return guard([&] {
    NONNULL(s);
    NONNULL(path);
    s->impl.save(path);
  });
}
hr_status hr_build_from_file(hr_store* s, const char* path, void* stream) {
  return guard([&] {
    NONNULL(s);
    NONNULL(path);
    s->impl.build_from_file(path, S(stream));
  });
}

hr_status hr_item_info(const hr_store* s, uint32_t item, uint32_t* scheme, uint32_t* tier, uint64_t* bytes) {
  return guard([&] {
    NONNULL(s);
    const auto& st = s->impl;
    harag::require(st.state != harag::Store::State::Empty, HR_ESTATE, "store not built");
    harag::require(item < st.n_items, HR_ENOTFOUND, "item id out of range");
    if (scheme) *scheme = st.scheme[item];
    if (tier) *tier = st.logical_tier(item);
    if (bytes) *bytes = st.bytes[item];
  });
}
hr_status hr_item_residency(const hr_store* s, uint32_t item, uint32_t* mask) {
  return guard([&] {
    NONNULL(s);
    NONNULL(mask);
    const auto& st = s->impl;
    harag::require(st.state != harag::Store::State::Empty, HR_ESTATE, "store not built");
    harag::require(item < st.n_items, HR_ENOTFOUND, "item id out of range");
    const auto& l = st.loc[item];
    const uint64_t none = harag::FreeList::kNone;
    *mask = (l.hbm_off != none ? HR_R_HBM : 0) | (l.pin_off != none ? HR_R_PIN : 0) |
            (l.page_off != none ? HR_R_PAGE : 0) | (l.backing_off != none ? HR_R_BACKING : 0) |
            (st.disk_fd >= 0 && !st.disk_off.empty() ? HR_R_FILE : 0);
  });
}
hr_status hr_store_local_cpus(const hr_store* s, int32_t* cpus, uint32_t cap, uint32_t* n) {
  return guard([&] {
    NONNULL(s);
    NONNULL(n);
    const auto& c = s->impl.local_cpus;
    *n = (uint32_t)c.size();
    harag::require(!cpus || c.size() <= cap, HR_EINVAL, "cpus buffer too small");
    for (size_t i = 0; cpus && i < c.size(); ++i) cpus[i] = c[i];
  });
}
hr_status hr_placement_hash(const hr_store* s, uint64_t* hash) {
  return guard([&] {
    NONNULL(s);
    NONNULL(hash);
    *hash = s->impl.placement_hash();
  });
}
hr_status hr_item_rank(const hr_store* s, uint32_t item, uint32_t* rank) {
  return guard([&] {
    NONNULL(s);
    NONNULL(rank);
    const auto& st = s->impl;
    harag::require(item < st.n_items, HR_ENOTFOUND, "item id out of range");
    for (uint32_t p = 0; p < st.n_items; ++p)
      if (st.order[p] == item) *rank = p;
  });
}
hr_status hr_export_item(const hr_store* s, uint32_t item, void* host_dst, size_t cap, size_t* len) {
  return guard([&] {
    NONNULL(s);
    NONNULL(host_dst);
    s->impl.export_item(item, host_dst, cap, len);
  });
}
hr_status hr_store_stats(const hr_store* s, hr_stats* out) {
  return guard([&] {
    NONNULL(s);
    NONNULL(out);
    const_cast<hr_store*>(s)->impl.get_stats(out);
  });
}
hr_status hr_set_timing(hr_store* s, int enable) {
  return guard([&] {
    NONNULL(s);
    harag::require(enable >= 0 && enable <= 3, HR_EINVAL, "enable must be 0..3");
    s->impl.timing = (enable & 1) != 0;
    s->impl.call_timing = (enable & 2) != 0;
  });
}
hr_status hr_last_call_ms(hr_store* s, double* ms) {
  return guard([&] {
    NONNULL(s);
    NONNULL(ms);
    *ms = s->impl.last_call_ms();
  });
}
hr_status hr_reset_stats(hr_store* s) {
  return guard([&] {
    NONNULL(s);
    hr_stats tmp;
    s->impl.get_stats(&tmp);
    s->impl.stats = hr_stats{};
  });
}

// ------------------------------------------------------------ host policy
hr_status hr_policy_rank(uint32_t n, const uint64_t* h, uint32_t* order_out) {
  return guard([&] {
    NONNULL(h);
    NONNULL(order_out);
    auto o = harag::rank_items(h, n);
    std::memcpy(order_out, o.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_policy_assign(uint32_t n, const uint64_t* h, uint32_t n_ladder, const uint32_t* ladder,
                           const double* tau, uint32_t* scheme_out) {
  return guard([&] {
    NONNULL(h);
    NONNULL(ladder);
    NONNULL(scheme_out);
    harag::require(n_ladder <= 1 || tau != nullptr, HR_EINVAL, "tau is NULL");
    auto sc = harag::assign_schemes(h, n, ladder, n_ladder, tau);
    std::memcpy(scheme_out, sc.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_policy_lists_bytes(uint32_t n, const uint32_t* order, const uint64_t* sizes, uint64_t hbm_budget,
                                uint64_t pin_budget, uint32_t* tier_out) {
  return guard([&] {
    NONNULL(order);
    NONNULL(sizes);
    NONNULL(tier_out);
    std::vector<uint32_t> o(order, order + n);
    for (uint32_t v : o) harag::require(v < n, HR_EINVAL, "order is not a permutation");
    auto t = harag::lists_by_bytes(o, sizes, hbm_budget, pin_budget);
    std::memcpy(tier_out, t.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_policy_lists_bytes4(uint32_t n, const uint32_t* order, const uint64_t* sizes, uint64_t hbm_budget,
                                 uint64_t pin_budget, uint64_t page_budget, uint32_t* tier_out) {
  return guard([&] {
    NONNULL(order);
    NONNULL(sizes);
    NONNULL(tier_out);
    std::vector<uint32_t> o(order, order + n);
    for (uint32_t v : o) harag::require(v < n, HR_EINVAL, "order is not a permutation");
    harag::require(page_budget != ~0ull, HR_EINVAL, "page_budget must be finite");
    auto t = harag::lists_by_bytes(o, sizes, hbm_budget, pin_budget, page_budget);
    std::memcpy(tier_out, t.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_policy_lists_fraction(uint32_t n, const uint32_t* order, double tau_gpu, double tau_pin,
                                   double tau_page, uint32_t* list_out) {
  return guard([&] {
    NONNULL(order);
    NONNULL(list_out);
    std::vector<uint32_t> o(order, order + n);
    for (uint32_t v : o) harag::require(v < n, HR_EINVAL, "order is not a permutation");
    auto l = harag::lists_by_fraction(o, tau_gpu, tau_pin, tau_page);
    std::memcpy(list_out, l.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_policy_count(uint32_t n_req, uint32_t k, const uint32_t* ids, uint32_t n_docs, uint64_t req_base,
                          uint32_t rank, uint32_t world, int64_t* delta_inout) {
  return guard([&] {
    NONNULL(ids);
    NONNULL(delta_inout);
    harag::count_requests(ids, n_req, k, n_docs, req_base, rank, world, delta_inout);
  });
}
hr_status hr_policy_epoch(uint32_t n, uint64_t* h_inout, const int64_t* delta, uint32_t decay_shift) {
  return guard([&] {
    NONNULL(h_inout);
    NONNULL(delta);
    harag::epoch_update(h_inout, delta, n, decay_shift);
  });
}
hr_status hr_item_bytes(const hr_store_config* cfg, uint32_t scheme, uint64_t* bytes) {
  return guard([&] {
    NONNULL(cfg);
    NONNULL(bytes);
    harag::require(scheme < HR_N_SCHEMES, HR_EINVAL, "unknown scheme");
    *bytes = harag::make_layout(*cfg).item_bytes(scheme);
  });
}

hr_status hr_exponent_histogram(uint32_t dtype, const void* src_dev, uint64_t n, uint64_t* hist_dev, void* stream) {
  return guard([&] {
    NONNULL(hist_dev);
    harag::require(dtype == HR_BF16 || dtype == HR_FP16, HR_EINVAL, "dtype must be HR_BF16 or HR_FP16");
    if (n == 0) return;
    NONNULL(src_dev);
    harag::launch_exponent_hist(dtype, src_dev, n, reinterpret_cast<unsigned long long*>(hist_dev), S(stream));
    HR_CUDA(cudaGetLastError());
  });
}

hr_status hr_guard_stats(const hr_store_config* cfg, const void* src_dev, uint64_t* stats_dev, void* stream) {
  return guard([&] {
    NONNULL(cfg);
    NONNULL(src_dev);
    NONNULL(stats_dev);
    harag::require(cfg->dtype == HR_BF16 || cfg->dtype == HR_FP16, HR_EINVAL, "dtype must be HR_BF16 or HR_FP16");
    harag::require(cfg->gse_ebits >= 2 && cfg->gse_mbits >= 2 && cfg->gse_ebits + cfg->gse_mbits == 7, HR_EINVAL,
                   "GSE-8 layout must be 1+e+m with e + m = 7, e, m >= 2");
    harag::launch_guard(cfg->dtype, src_dev, (uint64_t)cfg->L * cfg->H, (uint64_t)cfg->T * cfg->D, cfg->gse_ebits,
                        cfg->gse_mbits, reinterpret_cast<unsigned long long*>(stats_dev), S(stream));
  });
}
hr_status hr_policy_guard(uint32_t n, const uint32_t* schemes_in, const uint64_t* stats, uint32_t n_ladder,
                          const uint32_t* ladder, uint32_t* schemes_out) {
  return guard([&] {
    NONNULL(schemes_in);
    NONNULL(stats);
    NONNULL(ladder);
    NONNULL(schemes_out);
    auto sc = harag::guard_schemes(schemes_in, stats, n, ladder, n_ladder);
    std::memcpy(schemes_out, sc.data(), sizeof(uint32_t) * n);
  });
}
hr_status hr_scheme_error(const hr_store_config* cfg, uint32_t scheme, const void* src_dev, double* out_host,
                          void* stream) {
  return guard([&] {
    NONNULL(cfg);
    harag::scheme_error(*cfg, scheme, src_dev, out_host, S(stream));
  });
}

hr_status hr_alg2_create(uint32_t n_items, const uint32_t* list_of_item, const uint64_t* sizes, uint64_t cap_gpu,
                         uint64_t cap_pin, uint64_t cap_page, hr_alg2** out) {
  return guard([&] {
    NONNULL(list_of_item);
    NONNULL(out);
    *out = new hr_alg2(n_items, list_of_item, sizes, cap_gpu, cap_pin, cap_page);
  });
}
hr_status hr_alg2_access(hr_alg2* a, uint32_t item, uint32_t* hit_tier, uint32_t* put_mask, uint32_t* evicted,
                         uint32_t cap, uint32_t* n_evicted) {
  return guard([&] {
    NONNULL(a);
    auto o = a->impl.access(item);
    if (hit_tier) *hit_tier = o.hit;
    if (put_mask) *put_mask = o.put_mask;
    if (n_evicted) *n_evicted = (uint32_t)o.evicted.size();
    harag::require(o.evicted.size() <= cap || !evicted, HR_EINVAL, "evicted buffer too small");
    if (evicted)
      for (size_t i = 0; i < o.evicted.size(); ++i) evicted[i] = (o.evicted[i].first << 28) | o.evicted[i].second;
  });
}
hr_status hr_alg2_set_lists(hr_alg2* a, const uint32_t* list_of_item) {
  return guard([&] {
    NONNULL(a);
    NONNULL(list_of_item);
    a->impl.set_lists(list_of_item);
  });
}
hr_status hr_alg2_resident(const hr_alg2* a, uint32_t tier, uint32_t* items, uint32_t cap, uint32_t* n) {
  return guard([&] {
    NONNULL(a);
    NONNULL(n);
    auto r = a->impl.resident(tier);
    *n = (uint32_t)r.size();
    harag::require(!items || r.size() <= cap, HR_EINVAL, "items buffer too small");
    if (items) std::memcpy(items, r.data(), sizeof(uint32_t) * r.size());
  });
}
void hr_alg2_destroy(hr_alg2* a) { delete a; }

}  // extern "C"
