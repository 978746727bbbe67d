"""Oracle placement: Algorithm 2 (TEST INFRASTRUCTURE).

Tiers: GPU (HBM), PIN (pinned host), PAGE (pageable host), DISK (backing
store; here the library's pageable backing copy, R15/R16).
"""
from __future__ import annotations

import math
from collections import OrderedDict

from .hotness import rank_items

GPU, PIN, PAGE, DISK = "GPU", "PIN", "PAGE", "DISK"


def lists_by_fraction(order, tau_gpu: float, tau_pin: float, tau_page: float):
    """Alg. 2 step 1: split the hotness order into GPU_LIST,
    PIN_LIST, PAGE_LIST, DISK_LIST.  Fractions are paired with the list of the
    same name (R13; the printed line pairs idx_2 with tau_PAGE), floored
    (R11), and DISK_LIST ends at 2n exclusive (R14)."""
    M = len(order)
    i1 = math.floor(float(tau_gpu) * M)
    i2 = i1 + math.floor(float(tau_pin) * M)
    i3 = i2 + math.floor(float(tau_page) * M)
    if i3 > M:
        raise ValueError("fractions sum above 1")
    return list(order[:i1]), list(order[i1:i2]), list(order[i2:i3]), list(order[i3:])


def lists_by_bytes(order, sizes, hbm_budget: int, pin_budget: int):
    """Byte-budget variant of step 1 (R15): GPU_LIST is the longest rank-prefix
    whose item bytes fit hbm_budget; PIN_LIST the longest following run that
    fits pin_budget; the rest is PAGE_LIST (no skipping)."""
    gpu, pin, rest = [], [], []
    used = 0
    i = 0
    while i < len(order) and used + sizes[order[i]] <= hbm_budget:
        used += sizes[order[i]]
        gpu.append(order[i])
        i += 1
    used = 0
    while i < len(order) and used + sizes[order[i]] <= pin_budget:
        used += sizes[order[i]]
        pin.append(order[i])
        i += 1
    rest = list(order[i:])
    return gpu, pin, rest


def lists_by_bytes4(order, sizes, hbm_budget: int, pin_budget: int, page_budget: int):
    """Step 1 with all four lists of P:233-237 by bytes (R15, R26): GPU_LIST,
    PIN_LIST and PAGE_LIST are consecutive longest rank-prefixes fitting their
    budgets; DISK_LIST is the rest."""
    gpu, pin, rest = lists_by_bytes(order, sizes, hbm_budget, pin_budget)
    page, _, disk = lists_by_bytes(rest, sizes, page_budget, 0)
    return gpu, pin, page, disk


def eager_tiers(h, sizes, hbm_budget: int, pin_budget: int, backing_pinned: bool = False,
                page_budget=None):
    """Eager placement (R15): GPU_LIST resident in HBM, PIN_LIST in the pinned
    tier, the rest served from the backing (pageable, or pinned when the
    backing itself is pinned).  With page_budget (a disk-backed store, R26)
    PAGE_LIST is cached in pageable DRAM and DISK_LIST read from the file.
    Returns tier per item id."""
    order = rank_items(h)
    if page_budget is not None:
        gpu, pin, page, disk = lists_by_bytes4(order, sizes, hbm_budget, pin_budget, page_budget)
        tier = [None] * len(order)
        for lst, t in ((gpu, GPU), (pin, PIN), (page, PAGE), (disk, DISK)):
            for i in lst:
                tier[i] = t
        return tier
    if backing_pinned:
        pin_budget = 0
    gpu, pin, rest = lists_by_bytes(order, sizes, hbm_budget, pin_budget)
    tier = [None] * len(order)
    for i in gpu:
        tier[i] = GPU
    for i in pin:
        tier[i] = PIN
    for i in rest:
        tier[i] = PIN if backing_pinned else PAGE
    return tier


class LRUQueue:
    """A residency queue with capacity in bytes (count mode: every size 1).
    'Put with LRU': insert as most recent, evict least recently used
    until the queue fits (R16: LRU by last access in every tier)."""

    def __init__(self, capacity: int):
        self.capacity = int(capacity)
        self.q: OrderedDict[int, int] = OrderedDict()
        self.used = 0

    def __contains__(self, item) -> bool:
        return item in self.q

    def get(self, item) -> None:          # queue.get(C_i): refresh recency
        self.q.move_to_end(item)

    def put(self, item, size: int) -> list[int]:
        if item in self.q:
            self.q.move_to_end(item)
            return []
        if size > self.capacity:
            return []                     # cannot ever fit: not cached
        evicted = []
        while self.used + size > self.capacity:
            old, osz = self.q.popitem(last=False)
            self.used -= osz
            evicted.append(old)
        self.q[item] = size
        self.used += size
        return evicted


class Alg2:
    """Alg. 2 step 2, the demand-mode state machine.

    access(item) takes exactly one of the four branches and returns
    (hit_tier, puts, evictions) with puts = tiers the item was inserted into
    and evictions = [(tier, item)].  Promotion copies (inclusive, R16)."""

    def __init__(self, gpu_list, pin_list, page_list, caps, sizes=None):
        self.lists = (set(gpu_list), set(pin_list), set(page_list))
        self.sizes = sizes
        self.queues = {GPU: LRUQueue(caps[0]), PIN: LRUQueue(caps[1]), PAGE: LRUQueue(caps[2])}

    def _size(self, item) -> int:
        return 1 if self.sizes is None else int(self.sizes[item])

    def _put(self, tier, item, puts, ev):
        puts.append(tier)
        ev.extend((tier, e) for e in self.queues[tier].put(item, self._size(item)))

    def access(self, item):
        gl, pl, al = self.lists
        qg, qp, qa = self.queues[GPU], self.queues[PIN], self.queues[PAGE]
        puts, ev = [], []
        if item in qg:
            qg.get(item)
            return GPU, puts, ev
        if item in qp:
            qp.get(item)
            if item in gl:
                self._put(GPU, item, puts, ev)
            return PIN, puts, ev
        if item in qa:
            qa.get(item)
            if item in gl:
                self._put(GPU, item, puts, ev)
            if item in pl:
                self._put(PIN, item, puts, ev)
            return PAGE, puts, ev
        if item in gl:
            self._put(GPU, item, puts, ev)
        if item in pl:
            self._put(PIN, item, puts, ev)
        if item in al:
            self._put(PAGE, item, puts, ev)
        return DISK, puts, ev

    def set_lists(self, gpu_list, pin_list, page_list) -> None:
        """Re-placement in demand mode (R20): lists change, queues stay."""
        self.lists = (set(gpu_list), set(pin_list), set(page_list))

    def resident(self, tier) -> list[int]:
        return list(self.queues[tier].q.keys())
