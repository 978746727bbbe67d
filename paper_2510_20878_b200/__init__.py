"""B200-native HA-RAG hot path (arXiv 2510.20878): hotness-aware mixed-precision
KV-chunk store with a fused gather -> dequantise -> scatter assemble.

Thin Python layer over libharag.so (include/harag.h): argument marshalling
only.  Device memory, streams and process groups come from PyTorch; every step
of the path runs in the native library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (FP8E4M3, FP8E5M2, GSE8, HR_BF16, HR_FP16, INT4, INT8, MXFP8, PASS16, R_BACKING, R_FILE, R_HBM,
                   R_PAGE, R_PIN, SCHEMES, T_DISK, T_HBM, T_PAGE, T_PIN, HaragError, check, lib)

__all__ = ["Store", "HaragError", "SCHEMES", "PASS16", "INT8", "FP8E4M3", "FP8E5M2", "GSE8", "INT4", "MXFP8",
           "T_HBM", "T_PIN", "T_PAGE", "T_DISK", "R_HBM", "R_PIN", "R_PAGE", "R_BACKING", "R_FILE", "policy_rank", "policy_lists_bytes4", "policy_assign", "policy_lists_bytes",
           "policy_lists_fraction", "policy_count", "policy_epoch", "item_bytes", "Alg2",
           "exponent_histogram", "scheme_error", "guard_stats", "policy_guard"]


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def _stream(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def make_config(*, L, H, D, T, dtype="bf16", group=0, gse=(4, 3),
                ladder=("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), taus=(0.1, 0.1, 0.1),
                hbm_budget=0, pin_budget=0, backing_pinned=False, keep_backing=True, decay_shift=1,
                alias_R=0, device=0, rank=0, world=1, staging_slots=0, demand_mode=False,
                disk_backing=False, page_budget=0, numa_bind=True, guard=False) -> _lib.Config:
    c = _lib.default_config()
    c.L, c.H, c.D, c.T = L, H, D, T
    c.dtype = HR_FP16 if dtype == "fp16" else HR_BF16
    c.group = group
    c.gse_ebits, c.gse_mbits = gse
    if not 1 <= len(ladder) <= 6:
        raise ValueError("ladder must hold 1..6 schemes")
    if len(taus) != len(ladder) - 1:
        raise ValueError(f"need len(ladder) - 1 = {len(ladder) - 1} taus, got {len(taus)} (Alg. 1, P:190)")
    c.n_ladder = len(ladder)
    for j, s in enumerate(ladder):
        c.ladder[j] = SCHEMES[s] if isinstance(s, str) else int(s)
    for j, t in enumerate(taus):
        c.tau[j] = float(t)
    c.hbm_budget, c.pin_budget = int(hbm_budget), int(pin_budget)
    c.backing_pinned, c.keep_backing = int(backing_pinned), int(keep_backing)
    c.decay_shift, c.bench_alias_R = decay_shift, alias_R
    c.device, c.rank, c.world, c.staging_slots = device, rank, world, staging_slots
    c.demand_mode = int(bool(demand_mode))
    c.disk_backing = int(bool(disk_backing))
    c.page_budget = int(page_budget)
    c.numa_bind = int(bool(numa_bind))
    c.guard = int(bool(guard))
    return c


class _DevArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 2, "strides": None}


class Store:
    """One hr_store (one rank / GPU).  See include/harag.h for semantics."""

    def __init__(self, **cfg):
        self.cfg = make_config(**cfg)
        self._h = C.c_void_p()
        check(lib.hr_store_create(C.byref(self.cfg), C.byref(self._h)))
        self._keep = []

    # -------------------------------------------------------------- build
    def build(self, n_docs: int, hotness, source, stream=None) -> None:
        """source(doc, k_ptr, v_ptr, stream_handle) writes doc's K, V [L][H][T][D] on the device."""
        hot = _u64(hotness)

        def cb(user, doc, kp, vp, st):
            try:
                source(int(doc), int(kp), int(vp), int(st or 0))
                return 0
            except Exception:  # noqa: BLE001 - reported through the status code
                import traceback
                traceback.print_exc()
                return 1

        fn = _lib.SRC_FN(cb)
        check(lib.hr_build_store(self._h, n_docs, _p(hot, C.c_uint64), fn, None, _stream(stream)))

    def build_begin(self, n_docs: int, hotness, schemes=None) -> None:
        """hr_build_begin (Alg. 1), or hr_build_begin_schemes with the caller's per-item schemes."""
        hot = _u64(hotness)
        if schemes is None:
            check(lib.hr_build_begin(self._h, n_docs, _p(hot, C.c_uint64)))
        else:
            sc = _u32(schemes)
            check(lib.hr_build_begin_schemes(self._h, n_docs, _p(hot, C.c_uint64), _p(sc, C.c_uint32)))

    def build_put(self, doc: int, k_src, v_src, stream=None) -> None:
        check(lib.hr_build_put(self._h, doc, _ptr(k_src), _ptr(v_src), _stream(stream)))

    def build_put_batch(self, docs, k_srcs, v_srcs, stream=None) -> None:
        """hr_build_put_batch: up to 16 docs quantised in one launch."""
        n = len(docs)
        d = (C.c_uint32 * n)(*[int(x) for x in docs])
        ks = (C.c_void_p * n)(*[_ptr(x) for x in k_srcs])
        vs = (C.c_void_p * n)(*[_ptr(x) for x in v_srcs])
        check(lib.hr_build_put_batch(self._h, n, d, ks, vs, _stream(stream)))

    def build_end(self, stream=None) -> None:
        check(lib.hr_build_end(self._h, _stream(stream)))

    def save(self, path: str) -> None:
        """Persist the packed store (hr_store_save)."""
        check(lib.hr_store_save(self._h, str(path).encode()))

    def build_from_file(self, path: str, stream=None) -> None:
        """Build this (empty) store from a saved file (hr_build_from_file)."""
        check(lib.hr_build_from_file(self._h, str(path).encode(), _stream(stream)))

    # ----------------------------------------------------------- assemble
    def kv_bytes(self, k: int) -> int:
        return int(lib.hr_kv_bytes(self._h, k))

    def assemble(self, ids, k_out, v_out, stream=None) -> None:
        """ids uint32 [n_req][k]; k_out / v_out: sequences of device buffers (tensors or ints)."""
        ids = _u32(ids)
        if ids.ndim != 2:
            raise ValueError("ids must be [n_req][k]")
        n_req, k = ids.shape
        kp = (C.c_void_p * n_req)(*[_ptr(x) for x in k_out])
        vp = (C.c_void_p * n_req)(*[_ptr(x) for x in v_out])
        check(lib.hr_assemble_kv(self._h, n_req, k, _p(ids, C.c_uint32), kp, vp, _stream(stream)))

    def attend(self, ids, q, o, n_q: int, g: int, lse=None, scale: float = 0.0, kv_dump=None,
               stream=None, layers=None) -> None:
        """Attention of each request's query rows over its retrieved chunks, straight from the
        packed codes (hr_attend; hr_attend_layers for layers=(l0, n)).  q / o: device
        [n_req][L or n][Hl*g][n_q][D]; lse: device float32 [n_req][L or n][Hl*g][n_q] or None;
        scale <= 0 -> 1/sqrt(D)."""
        ids = _u32(ids)
        if ids.ndim != 2:
            raise ValueError("ids must be [n_req][k]")
        n_req, k = ids.shape
        if layers is None:
            check(lib.hr_attend(self._h, n_req, k, _p(ids, C.c_uint32), _ptr(q), int(n_q), int(g), _ptr(o),
                                _ptr(lse), float(scale), _ptr(kv_dump), _stream(stream)))
        else:
            check(lib.hr_attend_layers(self._h, n_req, k, _p(ids, C.c_uint32), int(layers[0]), int(layers[1]),
                                       _ptr(q), int(n_q), int(g), _ptr(o), _ptr(lse), float(scale),
                                       _ptr(kv_dump), _stream(stream)))

    def attend_prefill(self, ids, q, k_own, v_own, o, n_q: int, g: int, layers, lse=None, scale: float = 0.0,
                       stream=None) -> None:
        """hr_attend_prefill: chunk keys then the question's own keys (causal), layers=(l0, n);
        k_own / v_own: device [n_req][n][Hl][n_q][D]."""
        ids = _u32(ids)
        if ids.ndim != 2:
            raise ValueError("ids must be [n_req][k]")
        n_req, k = ids.shape
        check(lib.hr_attend_prefill(self._h, n_req, k, _p(ids, C.c_uint32), int(layers[0]), int(layers[1]), _ptr(q),
                                    _ptr(k_own), _ptr(v_own), int(n_q), int(g), _ptr(o), _ptr(lse), float(scale),
                                    _stream(stream)))

    # ------------------------------------------------------------ epochs
    def hotness_delta_ptr(self) -> tuple[int, int]:
        p = C.POINTER(C.c_int64)()
        n = C.c_uint32()
        check(lib.hr_hotness_delta(self._h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value or 0, int(n.value)

    def hotness_delta(self):
        """torch int64 tensor aliasing the store's device delta (for all_reduce)."""
        import torch
        ptr, n = self.hotness_delta_ptr()
        return torch.as_tensor(_DevArray(ptr, n, "<i8"), device=f"cuda:{self.cfg.device}")

    def replace(self, stream=None) -> None:
        check(lib.hr_replace(self._h, _stream(stream)))

    # -------------------------------------------------------- inspection
    def item_info(self, item: int) -> tuple[int, int, int]:
        s, t, b = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib.hr_item_info(self._h, item, C.byref(s), C.byref(t), C.byref(b)))
        return s.value, t.value, b.value

    def item_rank(self, item: int) -> int:
        r = C.c_uint32()
        check(lib.hr_item_rank(self._h, item, C.byref(r)))
        return r.value

    def item_residency(self, item: int) -> int:
        """Bit mask of the item's physical copies (hr_item_residency: R_HBM, R_PIN, R_PAGE, R_BACKING, R_FILE)."""
        m = C.c_uint32()
        check(lib.hr_item_residency(self._h, item, C.byref(m)))
        return m.value

    def local_cpus(self) -> list[int]:
        """CPUs the host tiers and bounce workers are bound to (hr_store_local_cpus; [] = unbound)."""
        buf = (C.c_int32 * 4096)()
        n = C.c_uint32()
        check(lib.hr_store_local_cpus(self._h, buf, 4096, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def placement_hash(self) -> int:
        """hr_placement_hash: digest of hotness, schemes and placement (compare across ranks)."""
        v = C.c_uint64()
        check(lib.hr_placement_hash(self._h, C.byref(v)))
        return v.value

    def export_item(self, item: int) -> np.ndarray:
        _, _, nbytes = self.item_info(item)
        buf = np.zeros(nbytes, dtype=np.uint8)
        ln = C.c_size_t()
        check(lib.hr_export_item(self._h, item, buf.ctypes.data, nbytes, C.byref(ln)))
        return buf[: ln.value]

    def set_timing(self, on: bool, calls: bool = False) -> None:
        """on: CUDA events around every assemble launch; calls: around every hr_assemble_kv call."""
        check(lib.hr_set_timing(self._h, int(bool(on)) | (2 if calls else 0)))

    def last_call_ms(self) -> float:
        """Device time of the last timed hr_assemble_kv call (entry -> last launch done)."""
        v = C.c_double()
        check(lib.hr_last_call_ms(self._h, C.byref(v)))
        return v.value

    def reset_stats(self) -> None:
        check(lib.hr_reset_stats(self._h))

    def stats(self) -> dict:
        s = _lib.Stats()
        check(lib.hr_store_stats(self._h, C.byref(s)))
        return {"requests": s.requests, "hits": list(s.hits), "bytes_out": s.bytes_out,
                "bytes_hbm_alg": s.bytes_hbm_alg, "bytes_h2d": s.bytes_h2d,
                "kernel_launches": s.kernel_launches, "migrations_in": s.migrations_in,
                "migrations_out": s.migrations_out, "failed_promotions": s.failed_promotions,
                "kernel_ms": s.kernel_ms, "timed_launches": s.timed_launches, "hbm_used": s.hbm_used,
                "pin_used": s.pin_used, "h2d_ms": s.h2d_ms, "h2d_items": s.h2d_items,
                "bytes_migrated": s.bytes_migrated, "hits_disk": s.hits_disk, "host_ms": s.host_ms,
                "quant_ms": s.quant_ms, "quant_launches": s.quant_launches}

    def close(self) -> None:
        if self._h:
            lib.hr_store_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


# ------------------------------------------------------------ host policy
def policy_rank(h) -> np.ndarray:
    h = _u64(h)
    out = np.empty(h.size, np.uint32)
    check(lib.hr_policy_rank(h.size, _p(h, C.c_uint64), _p(out, C.c_uint32)))
    return out


def policy_assign(h, ladder, taus) -> np.ndarray:
    h = _u64(h)
    if not 1 <= len(ladder) <= 6:
        raise ValueError("ladder must hold 1..6 schemes")
    if len(taus) != len(ladder) - 1:
        raise ValueError(f"need len(ladder) - 1 = {len(ladder) - 1} taus, got {len(taus)} (Alg. 1, P:190)")
    lad = _u32([SCHEMES[s] if isinstance(s, str) else s for s in ladder])
    tau = np.ascontiguousarray(np.asarray(list(taus) + [0.0], dtype=np.float64))
    out = np.empty(h.size, np.uint32)
    check(lib.hr_policy_assign(h.size, _p(h, C.c_uint64), lad.size, _p(lad, C.c_uint32),
                               _p(tau, C.c_double), _p(out, C.c_uint32)))
    return out


def policy_guard(schemes, stats, ladder) -> np.ndarray:
    """hr_policy_guard: stats = uint64 [n][2] as hr_guard_stats leaves them (flushed, fp32 bits of max |x|)."""
    sc, st = _u32(schemes), _u64(stats).reshape(-1)
    lad = _u32([SCHEMES[s] if isinstance(s, str) else s for s in ladder])
    out = np.empty(sc.size, np.uint32)
    check(lib.hr_policy_guard(sc.size, _p(sc, C.c_uint32), _p(st, C.c_uint64), lad.size, _p(lad, C.c_uint32),
                              _p(out, C.c_uint32)))
    return out


def guard_stats(src, stats, stream=None, **cfg) -> None:
    """hr_guard_stats: accumulate the guard statistics of one item's ALL-heads source [L][H][T][D] (device)
    into the device uint64[2] `stats` (zero it first); cfg as for Store (shape, dtype, gse)."""
    c = make_config(**cfg)
    check(lib.hr_guard_stats(C.byref(c), _ptr(src), _ptr(stats), _stream(stream)))


def policy_lists_bytes(order, sizes, hbm_budget, pin_budget) -> np.ndarray:
    o, s = _u32(order), _u64(sizes)
    out = np.empty(o.size, np.uint32)
    check(lib.hr_policy_lists_bytes(o.size, _p(o, C.c_uint32), _p(s, C.c_uint64), int(hbm_budget),
                                    int(pin_budget), _p(out, C.c_uint32)))
    return out


def policy_lists_bytes4(order, sizes, hbm_budget, pin_budget, page_budget) -> np.ndarray:
    o, s = _u32(order), _u64(sizes)
    out = np.empty(o.size, np.uint32)
    check(lib.hr_policy_lists_bytes4(o.size, _p(o, C.c_uint32), _p(s, C.c_uint64), int(hbm_budget),
                                     int(pin_budget), int(page_budget), _p(out, C.c_uint32)))
    return out


def policy_lists_fraction(order, tau_gpu, tau_pin, tau_page) -> np.ndarray:
    o = _u32(order)
    out = np.empty(o.size, np.uint32)
    check(lib.hr_policy_lists_fraction(o.size, _p(o, C.c_uint32), tau_gpu, tau_pin, tau_page,
                                       _p(out, C.c_uint32)))
    return out


def policy_count(ids, n_docs, req_base=0, rank=0, world=1, delta=None) -> np.ndarray:
    ids = _u32(ids)
    n_req, k = ids.shape
    d = np.zeros(2 * n_docs, np.int64) if delta is None else delta
    check(lib.hr_policy_count(n_req, k, _p(ids, C.c_uint32), n_docs, req_base, rank, world,
                              _p(d, C.c_int64)))
    return d


def policy_epoch(h, delta, decay_shift) -> np.ndarray:
    h = _u64(h).copy()
    dl = np.ascontiguousarray(np.asarray(delta, dtype=np.int64))
    check(lib.hr_policy_epoch(h.size, _p(h, C.c_uint64), _p(dl, C.c_int64), decay_shift))
    return h


def item_bytes(scheme, **cfg) -> int:
    c = make_config(**cfg)
    b = C.c_uint64()
    check(lib.hr_item_bytes(C.byref(c), SCHEMES[scheme] if isinstance(scheme, str) else scheme, C.byref(b)))
    return b.value


def exponent_histogram(src, n: int, dtype: str = "bf16", hist=None, stream=None):
    """hist[b] += count of the n 16-bit values at device address/tensor `src` whose biased
    exponent field is b.  `hist`: device uint64[256] (int64 tensor) to accumulate
    into; a fresh zeroed torch tensor on src's device when None (returned)."""
    if hist is None:
        import torch
        hist = torch.zeros(256, dtype=torch.int64, device=src.device)
    check(lib.hr_exponent_histogram(HR_BF16 if dtype == "bf16" else HR_FP16, _ptr(src), int(n), _ptr(hist),
                                    _stream(stream)))
    return hist


def scheme_error(scheme, src, stream=None, **cfg) -> tuple[float, float]:
    """(sum of squared errors, max |error|) of one item (device [L][H][T][D], this rank's heads)
    compressed with `scheme` and decoded by the assemble kernel — Eq. before the
    1/N and the square root.  Synchronous."""
    c = make_config(**cfg)
    out = (C.c_double * 2)()
    check(lib.hr_scheme_error(C.byref(c), SCHEMES[scheme] if isinstance(scheme, str) else scheme, _ptr(src), out,
                              _stream(stream)))
    return float(out[0]), float(out[1])


class Alg2:
    """Alg. 2 step 2 state machine: lists 0 GPU, 1 PIN, 2 PAGE, 3 DISK."""

    def __init__(self, list_of_item, caps, sizes=None):
        self.n = len(list_of_item)
        lst = _u32(list_of_item)
        sz = None if sizes is None else _u64(sizes)
        self._h = C.c_void_p()
        check(lib.hr_alg2_create(self.n, _p(lst, C.c_uint32), None if sz is None else _p(sz, C.c_uint64),
                                 int(caps[0]), int(caps[1]), int(caps[2]), C.byref(self._h)))

    def access(self, item: int):
        hit, mask, n = C.c_uint32(), C.c_uint32(), C.c_uint32()
        ev = (C.c_uint32 * max(1, self.n))()
        check(lib.hr_alg2_access(self._h, item, C.byref(hit), C.byref(mask), ev, max(1, self.n), C.byref(n)))
        return hit.value, mask.value, [(ev[i] >> 28, ev[i] & 0x0FFFFFFF) for i in range(n.value)]

    def set_lists(self, list_of_item) -> None:
        lst = _u32(list_of_item)
        check(lib.hr_alg2_set_lists(self._h, _p(lst, C.c_uint32)))

    def resident(self, tier: int) -> list[int]:
        n = C.c_uint32()
        buf = (C.c_uint32 * max(1, self.n))()
        check(lib.hr_alg2_resident(self._h, tier, buf, max(1, self.n), C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hr_alg2_destroy(self._h)
            self._h = None
