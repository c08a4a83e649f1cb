"""ORACLE -- test infrastructure, NOT part of the product.

A plain, slow, obviously-correct CPU implementation (NumPy fp64, pure-Python
loops where the definition is a loop) of what the EcoServe PaDG instance hot
path computes, written from the paper (PAPER.md, EcoServe sections) and
the readings listed in DESIGN.md section 3.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything under ``oracle/``. The product
(``paper_2504_18154_b200``, ``include/``, the CUDA library) never imports,
links or calls it, and the oracle never imports the product: the two share no
code. Only ``synthetic/`` (seeded input generators, no method arithmetic)
serves both.

Modules:
  transformer -- C1-C4: fp64 Llama-family forward, KV-cached decode, paged KV,
                 TP=2 partial sums (Eq. 1-3; Table 2).
  scheduler   -- C5: Alg. 1 InterSchedule and Alg. 2 CheckConstraints
                 (P:476-540, 556-567), the fixed integer cost model.
  des         -- C5: event-driven simulation of the intra-instance policy
                 (temporal disaggregation) and rolling
                 activation over a macro instance.
  tick_sim    -- brute-force fixed-tick simulator of the same semantics (pin).
  metrics     -- C6: TTFT / switch wait / TPOT (Sec. 3.3),
                 joint SLO attainment and goodput.
  accounting  -- Table 2 FLOP/byte expressions and KV bytes per token
                 (Table 3).
"""
