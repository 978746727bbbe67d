"""CPU oracle for the HA-RAG hot path (arxiv 2510.20878) — TEST INFRASTRUCTURE.

Plain, slow, obviously-correct numpy implementation of what the hot path
computes, written from /root/reference/PAPER.md (cited as ``P:<line>``) and,
where the paper is silent, from the readings listed in DESIGN.md §"Readings"
(cited as ``R<n>``).

ONLY ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product
(``paper_2510_20878_b200``, ``libharag.so``) never imports, links or calls it,
and this package imports nothing from the product: the two share no code.
The only common input is ``synth`` (seeded generators, no method arithmetic).

Modules
  numerics   bf16/fp16 <-> fp32 conversions (RNE by definition)
  codecs     INT8, INT4, FP8-E4M3, FP8-E5M2, GSE-8, PASS16 encode/decode
  hotness    access counting, Alg. 1 ranking + scheme assignment, epochs
  placement  Alg. 2 lists, byte-budget lists, the demand-mode state machine
  store      packed item blob format, build, assemble (per-request KV layout)

Floating point: every decision the method takes in floating point (scales,
quantised codes) is taken in IEEE fp32 with round-to-nearest-even, one
operation at a time (numpy never contracts), because the product computes in
fp32 and "where floating point decides an integer, both sides take that
decision in the same precision" (R3).  Exact quantities (FP8 and
GSE-8 decoded values, distances for nearest-code search) are computed in fp64,
where they are exact.

Pinning: tests/test_oracle_*.py check this package against values the paper
prints (P:172 shared-exponent array), SPEC.md worked examples, exhaustive
sweeps, closed forms, brute force on tiny inputs and library routines
(ml_dtypes / torch float8 casts).  Functions without such a pin say
"parity unpinned" below; currently: none of the arithmetic; the 1+4+3 layout
*preference* of P:327 is an empirical claim, not a function, and is unpinned.
"""
