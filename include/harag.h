/*
 * harag.h — C ABI of the B200-native HA-RAG hot path (arXiv 2510.20878).
 *
 * "build_store(chunks, hotness) -> quantised store + placement" and
 * "assemble_kv(request chunk ids) -> KV cache", plus hotness update and
 * re-placement (BASELINE.json north_star).  Paper citations are
 * /root/reference/PAPER.md line numbers (P:<line>); readings R<n> are the
 * numbered rows of DESIGN.md §2.
 *
 * Conventions
 *  - Plain C: fixed-width integers, plain pointers, sizes in bytes.  CUDA
 *    streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 *    default stream).  Device pointers are CUDA device addresses on the
 *    store's device.
 *  - Every function returns hr_status; on failure hr_last_error() returns a
 *    thread-local message.  Validation errors (HR_EINVAL, HR_ENOTFOUND) are
 *    returned BEFORE any device work is enqueued: no partial writes.
 *  - No C++ exception crosses the ABI.
 *  - A store is single-writer: calls on one store must be serialised by the
 *    caller.  Different stores (one per rank/GPU) are independent.
 *  - Ownership: the store owns every buffer it allocates (HBM arena, pinned
 *    tier, host backing, staging ring, descriptor buffers, the per-doc source
 *    buffers handed to hr_src_fn).  The caller owns inputs and outputs.
 *
 * Item numbering: item = 2*doc + kind, kind 0 = K, 1 = V — the paper's 2n
 * chunks [C_1^k, C_1^v, ..., C_n^k, C_n^v] (Alg. 1 input).
 */
#ifndef HARAG_H
#define HARAG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HR_ABI_VERSION 2

typedef enum {
  HR_OK = 0,
  HR_EINVAL = 1,     /* bad argument: shape, tau out of range, duplicate id in a request, NaN/Inf source */
  HR_ENOMEM = 2,     /* device or host allocation failed */
  HR_ECUDA = 3,      /* a CUDA runtime call failed (message has the CUDA error string) */
  HR_ENOTFOUND = 4,  /* unknown doc / item id */
  HR_ECORRUPT = 5,   /* malformed packed data (e.g. GSE-8 index past the array) */
  HR_ESTATE = 6      /* call not valid in the store's current state (e.g. assemble before build) */
} hr_status;

typedef enum { HR_BF16 = 0, HR_FP16 = 1 } hr_dtype;   /* source dtype == output dtype */

/* Compression schemes S_i of Alg. 1 plus the north_star 16-bit
 * passthrough and INT4.  P:397: INT8 -> E4M3 -> E5M2 -> GSE-8 hottest to coldest. */
typedef enum {
  HR_S_PASS16 = 0,   /* source bits unchanged (byte-identical tier) */
  HR_S_INT8 = 1,     /* P:144; symmetric per-group absmax, codes [-127,127] (R1-R3) */
  HR_S_FP8E4M3 = 2,  /* P:144; RNE, saturating at 448 (R5) */
  HR_S_FP8E5M2 = 3,  /* P:144; RNE, saturating at 57344 (R5) */
  HR_S_GSE8 = 4,     /* P:155-172; 1+e+m grouped shared exponent, per-slab array (R6-R9) */
  HR_S_INT4 = 5,     /* north_star; per-group min-max, two codes per byte (R4) */
  HR_S_MXFP8 = 6     /* Blackwell-style microscaling — E8M0 scale per 32 elements,
                        E4M3 elements (R31); not in the paper's ladder, usable in any ladder */
} hr_scheme;
#define HR_N_SCHEMES 7

typedef enum {
  HR_T_HBM = 0,      /* GPU memory (queueGPU) */
  HR_T_PIN = 1,      /* pinned host memory (queuePIN) */
  HR_T_PAGE = 2,     /* pageable host memory (queuePAGE / in-memory backing store) */
  HR_T_DISK = 3      /* the store file only (disk_backing; DISK_LIST) */
} hr_tier;

typedef struct {
  /* model KV shape: L layers, H KV heads, D head_dim, T tokens per chunk (512) */
  uint32_t L, H, D, T;
  uint32_t dtype;          /* hr_dtype */
  uint32_t group;          /* INT8/INT4 group G in elements (0 -> D); power of two, 32 <= G, G | T*D (R1) */
  uint32_t gse_ebits;      /* GSE-8 layout 1+e+m, e+m = 7, e,m >= 2 (default 4,3) */
  uint32_t gse_mbits;
  uint32_t n_ladder;       /* 1..6 schemes, hottest first (Alg. 1 S_1..S_m) */
  uint32_t ladder[6];      /* hr_scheme */
  double   tau[6];         /* tau[0..n_ladder-2]: fractions of the 2n items per group; the last group takes the remainder (R11) */
  uint64_t hbm_budget;     /* bytes of HBM arena per rank (GPU_LIST capacity, R15) */
  uint64_t pin_budget;     /* bytes of pinned host tier per rank (PIN_LIST capacity) */
  int32_t  backing_pinned; /* 1: host backing is pinned (every non-HBM item is served as PIN); 0: pageable */
  int32_t  keep_backing;   /* 1: every item keeps a host backing copy (needed by hr_replace); 0: HBM items live only in HBM */
  int32_t  demand_mode;    /* 0: eager placement (GPU_LIST / PIN_LIST resident after build and after each hr_replace);
                              1: paper-literal Alg. 2 step 2: queues start empty, every access takes one
                              branch, promotes inclusively with LRU (R16); forces keep_backing = 1 */
  uint32_t decay_shift;    /* epoch: h <- (h >> decay_shift) + delta (R20) */
  uint32_t bench_alias_R;  /* 0 = off; >0: docs d and d' with d % R == d' % R and equal scheme share one host backing blob (bench only) */
  int32_t  device;         /* CUDA device ordinal */
  int32_t  rank, world;    /* this store owns KV heads [rank*H/world, (rank+1)*H/world) */
  uint32_t staging_slots;  /* host-tier staging ring slots in HBM, one item each (0 -> ~2 GiB worth, 3..128) */
  int32_t  disk_backing;   /* stores built with hr_build_from_file only: 1 = items outside the HBM arena and the
                              pinned tier stay in the file and are read on every miss (the paper's DISK tier,
                              P:237; O_DIRECT when available); 0 = the file is loaded into host memory */
  uint64_t page_budget;    /* disk_backing only: bytes of pageable cache for PAGE_LIST items (queuePAGE);
                              items past GPU_LIST + PIN_LIST + PAGE_LIST are DISK_LIST (read on every miss) */
  int32_t  numa_bind;      /* 1 (default): host tiers (pinned tier, backing, bounce buffers) are allocated and
                              first touched by a thread running on the CPUs NVML reports local to `device`, and
                              the bounce / disk workers run there (hr_store_local_cpus); 0: no binding */
  int32_t  guard;          /* hr_build_store only: 1 = value-distribution guard (R29, an extension the
                              paper does not have): before placement, every item whose Alg. 1 scheme would lose
                              values (GSE-8 flushing nonzeros to 0, FP8 saturating) moves up the ladder
                              (hr_guard_stats, hr_policy_guard); 0 (default) = Alg. 1 as published */
} hr_store_config;

typedef struct {
  uint64_t requests;          /* requests assembled */
  uint64_t hits[3];           /* item accesses served per hr_tier */
  uint64_t bytes_out;         /* assembled KV bytes written */
  uint64_t bytes_hbm_alg;     /* algorithmic HBM bytes of the assemble kernels (codes+meta read, out written) */
  uint64_t bytes_h2d;         /* host -> device bytes moved by the streamer */
  uint64_t kernel_launches;   /* assemble kernel launches */
  uint64_t migrations_in;     /* items promoted into HBM by hr_replace */
  uint64_t migrations_out;    /* items evicted from HBM by hr_replace */
  uint64_t failed_promotions; /* promotions that found no contiguous arena space */
  double   kernel_ms;         /* sum of assemble-kernel durations (CUDA events) when timing is on */
  uint64_t timed_launches;    /* launches included in kernel_ms */
  uint64_t hbm_used;          /* bytes of HBM arena in use */
  uint64_t pin_used;          /* bytes of pinned tier in use */
  double   h2d_ms;            /* sum over assemble calls of the host->device copy window (first copy start ->
                                 last copy end, CUDA events on the copy stream) when timing is on */
  uint64_t h2d_items;         /* host-tier items streamed */
  uint64_t bytes_migrated;    /* host -> device bytes of hr_replace promotions (not in bytes_h2d) */
  uint64_t hits_disk;         /* item accesses served from the store file (HR_T_DISK) */
  double   host_ms;           /* host time inside hr_assemble_kv (entry -> last launch enqueued), summed */
  double   quant_ms;          /* sum of quantize-launch durations (CUDA events) of hr_build_put* when timing is on */
  uint64_t quant_launches;    /* quantize launches included in quant_ms */
} hr_stats;

typedef struct hr_store hr_store;
typedef struct hr_alg2 hr_alg2;

/* Source of one document's K and V chunks for hr_build_store: write them as
 * [L][H][T][D] (ALL heads, source dtype) into the library-owned DEVICE
 * buffers k_dst / v_dst, ordered on `stream`.  Return HR_OK or an error that
 * aborts the build. */
typedef int (*hr_src_fn)(void* user, uint32_t doc, void* k_dst, void* v_dst, void* stream);

/* ---------------------------------------------------------------- basics */
const char* hr_last_error(void);             /* thread-local message of the last failure ("" if none) */
uint32_t    hr_abi_version(void);            /* HR_ABI_VERSION */
void        hr_config_default(hr_store_config* cfg);  /* paper defaults: ladder INT8,E4M3,E5M2,GSE8 at tau 10/10/10%, GSE 1+4+3, bf16 */

/* Create an empty store on cfg->device.  Validates the shape (D % 8 == 0,
 * T*D % 256 == 0, H % world == 0, group rules), ladder and taus (HR_EINVAL).
 * Allocates nothing large until hr_build_begin. */
hr_status hr_store_create(const hr_store_config* cfg, hr_store** out);
void      hr_store_destroy(hr_store* s);     /* frees everything; NULL is a no-op; synchronises the device */

/* ------------------------------------------------------------------ build
 * Alg. 1: rank items by hotness (desc, ties by id, R12), give
 * group j scheme ladder[j]; then quantise every item (a3/a4) and place it
 * (Alg. 2 step 1 by bytes, R15): GPU_LIST -> HBM arena, PIN_LIST -> pinned
 * tier, the rest -> host backing.
 *   hotness: host uint64[2*n_docs], the access-frequency vector AF. */
hr_status hr_build_store(hr_store* s, uint32_t n_docs, const uint64_t* hotness,
                         hr_src_fn src, void* user, void* stream);

/* The same build in three calls: begin (ranking, schemes, placement,
 * allocations), put (quantise one doc from caller-owned DEVICE buffers k_src,
 * v_src, each [L][H][T][D] all heads, source dtype; they are read on
 * `stream`, so the caller keeps them alive until the stream passes this
 * point), end (synchronise; every doc must have been put and no NaN/Inf
 * seen, else HR_EINVAL). */
hr_status hr_build_begin(hr_store* s, uint32_t n_docs, const uint64_t* hotness);
/* hr_build_begin with the caller's schemes (host uint32[2*n_docs], each one of cfg->ladder) in place of
 * Alg. 1's — e.g. hr_policy_guard's; placement still ranks by `hotness`.  HR_EINVAL for a scheme
 * outside the ladder. */
hr_status hr_build_begin_schemes(hr_store* s, uint32_t n_docs, const uint64_t* hotness, const uint32_t* schemes);
hr_status hr_build_put(hr_store* s, uint32_t doc, const void* k_src, const void* v_src, void* stream);
/* hr_build_put for n <= 16 distinct docs in one quantize launch (all 2n items, any scheme mix):
 * docs host uint32[n], k_srcs / v_srcs host arrays of n DEVICE pointers (same rules as hr_build_put).
 * HR_EINVAL for n > 16, a NULL pointer or a repeated doc; HR_ENOTFOUND for a doc >= n_docs; checks
 * precede any launch. */
hr_status hr_build_put_batch(hr_store* s, uint32_t n, const uint32_t* docs, const void* const* k_srcs,
                             const void* const* v_srcs, void* stream);
hr_status hr_build_end(hr_store* s, void* stream);

/* --------------------------------------------------------------- assemble
 * a6-a8: for each request r (n_req requests of k DISTINCT doc ids, host
 * uint32 [n_req][k], copied at call time) write this rank's heads of
 *   K_out[r][l][h][j*T + t][d] = dequant(item 2*doc_{r,j})[l][h][t][d]
 *   V_out[r][l][h][j*T + t][d] = dequant(item 2*doc_{r,j}+1)[l][h][t][d]
 * into k_out[r] / v_out[r] (DEVICE pointers, each hr_kv_bytes(s,k) bytes,
 * 16-B aligned, source dtype, RNE — R25).  HBM-resident items are decoded
 * in place; host-tier items are streamed through the staging ring first
 * (pageable -> pinned bounce -> HBM).  Also counts hotness (a1): each
 * request q (running count over the store's life) with q % world == rank
 * adds 1 to both items of each of its docs in the device delta vector.
 * Stream-ordered: outputs are valid when `stream` reaches this point.
 * Errors: unknown doc -> HR_ENOTFOUND; duplicate doc in one request or k == 0
 * -> HR_EINVAL (R19); before build -> HR_ESTATE. */
size_t    hr_kv_bytes(const hr_store* s, uint32_t k);   /* bytes of ONE of K/V for k docs on this rank */
hr_status hr_assemble_kv(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids,
                         void* const* k_out, void* const* v_out, void* stream);

/* ------------------------------------------------------- hotness / epochs
 * a9 (R20).  hr_hotness_delta exposes the store's DEVICE int64[2*n_docs]
 * per-item access counts since the last hr_replace (for an in-place
 * torch.distributed.all_reduce(SUM) across ranks).  hr_replace consumes the
 * (reduced) delta: h <- (h >> decay_shift) + delta, re-rank, recompute the
 * GPU/PIN lists (schemes stay fixed: compress once), evict items that
 * left GPU_LIST and promote the newcomers (H2D from the host backing; needs
 * keep_backing = 1, else HR_ESTATE), zero the delta.  Synchronises `stream`
 * once to read the delta; promotions are asynchronous (an item is served from
 * the host until its copy lands) and are ordered after all work already
 * enqueued on `stream` — callers that assemble on several streams must
 * synchronise the others first.  Demand mode: only the lists change. */
hr_status hr_hotness_delta(hr_store* s, int64_t** dev_ptr, uint32_t* n);
hr_status hr_replace(hr_store* s, void* stream);

/* Consumer of the assembled KV: for each request r the
 * attention of its query rows over its k retrieved chunks — the cross-attention
 * a TurboRAG / HA-RAG prefill runs over the precomputed chunk KV —
 * computed straight from the packed codes (gather + dequantise fused into the
 * kernel; the KV cache of hr_assemble_kv is never materialised):
 *   O[r][l][hq][i][:] = sum_j softmax_j(scale * <Q[r][l][hq][i], K_j>) V_j,
 *   lse[r][l][hq][i]  = log sum_j exp(scale * <Q[r][l][hq][i], K_j>)  (natural log),
 * j over the k*T keys of docs ids[r][0..k) in request order, K_j / V_j the
 * decoded values of hr_assemble_kv (bit for bit), query head hq of this rank
 * reading local KV head hq / g (GQA).
 *   q_dev:   device [n_req][L][Hl*g][n_q][D] of cfg->dtype (16-byte aligned);
 *   o_dev:   device, same layout and dtype; lse_dev: device float32
 *            [n_req][L][Hl*g][n_q], or NULL;
 *   scale:   softmax scale (<= 0 -> 1/sqrt(D));
 *   kv_dump: NULL (test hook: device [n_req][2][L][Hl][k*T][D], receives the
 *            decoded K and V exactly as hr_assemble_kv would write them).
 * Needs g * n_q <= 128, D in {64, 128}, T a multiple of 64 and eager placement (HR_ESTATE otherwise,
 * before any launch); host-tier items are staged as in hr_attend_layers;
 * duplicate / unknown ids as hr_assemble_kv.  Stream-ordered; counts hotness
 * like hr_assemble_kv (a1).  Arithmetic: bf16/fp16 tensor-core products, fp32
 * accumulation, probabilities rounded to the dtype before P.V.
 * A call whose (request, layer, KV head) units alone leave SMs idle splits each
 * unit's keys over several CTAs and merges the partial results by LSE (a
 * store-owned workspace; successive split launches are ordered by an event,
 * also across streams; HARAG_ATT_SPLIT forces a split count). */
hr_status hr_attend(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, const void* q_dev,
                    uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev, float scale, void* kv_dump,
                    void* stream);
/* hr_attend over the layer window [layer0, layer0 + n_layers) only — one layer at a time is what a
 * prefill needs, since layer l's queries come out of layer l-1.  q_dev / o_dev / lse_dev / kv_dump are
 * laid out as for hr_attend with n_layers in place of L.  Items outside the HBM arena are accepted:
 * the window's code and meta slabs are copied from the pinned tier / host backing (pageable through a
 * pinned bounce; the DISK tier through a read of the blob) into staging-ring slots, and the
 * launch waits for them; a call's host-tier items must fit the ring at once (HR_ESTATE otherwise,
 * before any work).  hr_attend == hr_attend_layers(s, ..., 0, L, ...). */
hr_status hr_attend_layers(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, uint32_t layer0,
                           uint32_t n_layers, const void* q_dev, uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev,
                           float scale, void* kv_dump, void* stream);

/* hr_attend_layers in the prefill form (R30; TurboRAG prefill): the question's
 * own keys and values follow the chunk keys and are attended causally — query row (hq, i) (question
 * token i) sees every chunk key and own keys 0..i — so O / LSE are the full prefill attention of the
 * question tokens over [retrieved chunk KV ; question KV] in one launch.
 *   k_own_dev, v_own_dev: device [n_req][n_layers][Hl][n_q][D] of cfg->dtype (this rank's KV heads,
 *                         K already position-encoded), 16-byte aligned;
 *   everything else as hr_attend_layers (no kv_dump); needs n_q <= 64 and k <= 63 (HR_EINVAL). */
hr_status hr_attend_prefill(hr_store* s, uint32_t n_req, uint32_t k, const uint32_t* doc_ids, uint32_t layer0,
                            uint32_t n_layers, const void* q_dev, const void* k_own_dev, const void* v_own_dev,
                            uint32_t n_q, uint32_t g, void* o_dev, float* lse_dev, float scale, void* stream);

/* ------------------------------------------------------------ persistence
 * Compress once, load many (compressed chunks are stored on disk).
 * hr_store_save writes a built store: a 4 KiB-aligned header (magic
 * "HRSTORE1", the config, n_docs, per-item hotness and scheme) followed by
 * every item's packed blob at a 4 KiB-aligned offset.
 * Synchronous; HR_ECUDA/HR_EINVAL (I/O errors carry errno text).
 * hr_build_from_file builds an EMPTY store from such a file instead of
 * quantising: schemes are the saved ones (compress once), hotness the saved
 * vector, placement (Alg. 2 step 1) follows this store's budgets.  The file's
 * shape (L, H, D, T, dtype, group, GSE layout, rank, world) must equal the
 * store's config, else HR_EINVAL.  With disk_backing = 1 the file stays open
 * and backs the cold items. */
hr_status hr_store_save(const hr_store* s, const char* path);
hr_status hr_build_from_file(hr_store* s, const char* path, void* stream);

/* ------------------------------------------------------------- inspection */
/* tier: eager mode -> where the item is served from (HBM arena, pinned tier, backing);
 * demand mode -> the Alg. 2 queue holding it (queueGPU -> HBM, queuePIN -> PIN, none -> PAGE/backing). */
hr_status hr_item_info(const hr_store* s, uint32_t item, uint32_t* scheme, uint32_t* tier, uint64_t* bytes);
hr_status hr_item_rank(const hr_store* s, uint32_t item, uint32_t* rank);   /* position in the hotness order */
/* Physical copies of an item right now (hr_item_info reports the logical tier): *mask |= HR_R_HBM when
 * the item's blob is in the HBM arena (or its promotion copy is enqueued there; stream-ordered), HR_R_PIN
 * pinned-tier copy, HR_R_PAGE pageable PAGE-tier cache copy, HR_R_BACKING in-memory host backing,
 * HR_R_FILE in the store file of a disk-backed store.  Demand mode keeps HR_R_HBM == queueGPU of Alg. 2
 * after every hr_assemble_kv.  HR_ENOTFOUND for an unknown item, HR_ESTATE before build. */
enum { HR_R_HBM = 1, HR_R_PIN = 2, HR_R_PAGE = 4, HR_R_BACKING = 8, HR_R_FILE = 16 };
hr_status hr_item_residency(const hr_store* s, uint32_t item, uint32_t* mask);
/* CPUs the store binds its host-tier allocations and workers to (numa_bind): *n of them written to
 * cpus[0..cap); *n = 0 when nothing is bound (no NVML, numa_bind = 0, or every allowed CPU is local). */
hr_status hr_store_local_cpus(const hr_store* s, int32_t* cpus, uint32_t cap, uint32_t* n);
/* Digest of the placement state every rank must agree on after an epoch (SURVEY §8(e) consistency
 * check): FNV-1a over, per item in id order, its hotness h, scheme and target tier (eager) / queue
 * (demand mode), and over the hotness rank order.  Ranks of one job compare it with a MIN/MAX
 * all-reduce; a mismatch means their hotness vectors or policies diverged. */
hr_status hr_placement_hash(const hr_store* s, uint64_t* hash);
hr_status hr_export_item(const hr_store* s, uint32_t item, void* host_dst, size_t cap, size_t* len); /* packed blob; synchronous */
hr_status hr_store_stats(const hr_store* s, hr_stats* out);                 /* synchronises pending timing events */
hr_status hr_set_timing(hr_store* s, int enable);  /* bit 0: time every assemble launch with CUDA events (stats.kernel_ms);
                                                     bit 1: time every hr_assemble_kv call (hr_last_call_ms); 0..3 */
/* Per-request assemble latency: device time from the entry of the last hr_assemble_kv call made with
 * timing bit 1 (an event recorded on its stream before any of its work) to the end of its last launch —
 * planning, descriptor upload, host-tier copies and kernels included.  Waits for that call to finish.
 * HR_ESTATE when no call was timed. */
hr_status hr_last_call_ms(hr_store* s, double* ms);
hr_status hr_reset_stats(hr_store* s);

/* ------------------------------------------ host policy (no GPU needed)
 * The same C++ code the store uses, exposed for host-side tests and tools. */
/* Alg. 1 line 1: order_out = item ids by (h desc, id asc). */
hr_status hr_policy_rank(uint32_t n_items, const uint64_t* h, uint32_t* order_out);
/* Alg. 1: scheme per item. */
hr_status hr_policy_assign(uint32_t n_items, const uint64_t* h, uint32_t n_ladder, const uint32_t* ladder,
                           const double* tau, uint32_t* scheme_out);
/* Alg. 2 step 1 by bytes (R15): tier per item (0 HBM, 1 PIN, 2 PAGE). */
hr_status hr_policy_lists_bytes(uint32_t n_items, const uint32_t* order, const uint64_t* sizes,
                                uint64_t hbm_budget, uint64_t pin_budget, uint32_t* tier_out);
/* The same with a PAGE budget: 0 HBM, 1 PIN, 2 PAGE, 3 DISK (the rest). */
hr_status hr_policy_lists_bytes4(uint32_t n_items, const uint32_t* order, const uint64_t* sizes,
                                 uint64_t hbm_budget, uint64_t pin_budget, uint64_t page_budget, uint32_t* tier_out);
/* Alg. 2 step 1 by fractions (R13, R14): list per item (0 GPU, 1 PIN, 2 PAGE, 3 DISK). */
hr_status hr_policy_lists_fraction(uint32_t n_items, const uint32_t* order, double tau_gpu, double tau_pin,
                                   double tau_page, uint32_t* list_out);
/* a1 on the host: delta[2*doc+kind] += 1 for requests q = req_base + r with q % world == rank. */
hr_status hr_policy_count(uint32_t n_req, uint32_t k, const uint32_t* ids, uint32_t n_docs, uint64_t req_base,
                          uint32_t rank, uint32_t world, int64_t* delta_inout);
/* a9: h <- (h >> decay_shift) + delta (negative results -> HR_EINVAL). */
hr_status hr_policy_epoch(uint32_t n_items, uint64_t* h_inout, const int64_t* delta, uint32_t decay_shift);
/* Packed blob size of one item for a config and scheme. */
hr_status hr_item_bytes(const hr_store_config* cfg, uint32_t scheme, uint64_t* bytes);

/* ---- analysis tooling -------------------------------
 * hr_exponent_histogram: hist_dev[b] += number of the n 16-bit values at src_dev
 * (device, dtype hr_dtype) whose biased exponent field is b (bf16: bits 14..7,
 * 256 bins; fp16: bits 14..10, 32 bins used) — the exponent distribution of
 * P:131-133 (Fig. KV-exponent-range); zeros/subnormals land in bin 0.
 * hist_dev: device uint64[256], accumulated (the caller zeroes it).  Stream-
 * ordered; src_dev 16-byte aligned for full speed (any alignment is correct). */
hr_status hr_exponent_histogram(uint32_t dtype, const void* src_dev, uint64_t n, uint64_t* hist_dev, void* stream);
/* hr_scheme_error: compress one item with `scheme` exactly as hr_build_store
 * would (cfg's geometry, group, GSE layout and this rank's heads of src_dev,
 * device [L][H][T][D] of cfg->dtype), decode it with the assemble kernel, and
 * write out_host[0] = sum over elements of (x_i - x^_i)^2 (fp64), out_host[1] =
 * max |x_i - x^_i|; RMSE of Eq. = sqrt(out_host[0] / (L*Hl*T*D)).
 * Synchronous (returns after the stream drains).  HR_EINVAL on NaN/Inf input or
 * a bad config / scheme; temporary device memory is freed before returning. */
/* Value-distribution guard statistics of one item (R29): src_dev =
 * the item's source [L][H][T][D] over ALL heads (so every rank of a head-sharded store derives the same
 * schemes), dtype / layout from cfg.  Accumulates into DEVICE stats_dev[2]: [0] += the values GSE-8
 * (cfg's 1+e+m layout, each (layer, head) slab with its own rule-C array) would flush to zero —
 * nonzero fp32 subnormals and exponents below G_0 - (m-1) (R9); [1] = max([1], fp32 bits of max |x|).
 * Zero stats_dev before the first call of an item.  Stream-ordered. */
hr_status hr_guard_stats(const hr_store_config* cfg, const void* src_dev, uint64_t* stats_dev, void* stream);
/* The guard's policy: for item i with Alg. 1 scheme schemes_in[i] and stats[2i], stats[2i+1] (host, as
 * hr_guard_stats leaves them), while the scheme would lose values (GSE-8: any flushed value; FP8 E4M3:
 * max |x| > 448; E5M2: > 57344, R5) and is not ladder[0], take the previous (hotter) ladder scheme.
 * HR_EINVAL for a scheme outside the ladder. */
hr_status hr_policy_guard(uint32_t n_items, const uint32_t* schemes_in, const uint64_t* stats, uint32_t n_ladder,
                          const uint32_t* ladder, uint32_t* schemes_out);
hr_status hr_scheme_error(const hr_store_config* cfg, uint32_t scheme, const void* src_dev, double* out_host,
                          void* stream);

/* Alg. 2 step 2 demand-mode state machine.  list_of_item: 0 GPU,
 * 1 PIN, 2 PAGE, 3 DISK; sizes: bytes per item (NULL = 1 each); caps in the
 * same unit.  access(): hit_tier 0 GPU / 1 PIN / 2 PAGE / 3 DISK; put_mask bit
 * t = inserted into tier t; evicted[0..*n_evicted) = (tier << 28 | item)
 * (cap entries, HR_EINVAL if too small).  Inclusive promotion, LRU (R16). */
hr_status hr_alg2_create(uint32_t n_items, const uint32_t* list_of_item, const uint64_t* sizes,
                         uint64_t cap_gpu, uint64_t cap_pin, uint64_t cap_page, hr_alg2** out);
hr_status hr_alg2_access(hr_alg2* a, uint32_t item, uint32_t* hit_tier, uint32_t* put_mask,
                         uint32_t* evicted, uint32_t cap, uint32_t* n_evicted);
hr_status hr_alg2_set_lists(hr_alg2* a, const uint32_t* list_of_item);
hr_status hr_alg2_resident(const hr_alg2* a, uint32_t tier, uint32_t* items, uint32_t cap, uint32_t* n);
void      hr_alg2_destroy(hr_alg2* a);

#ifdef __cplusplus
}
#endif
#endif /* HARAG_H */
