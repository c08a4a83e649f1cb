"""Seeded synthetic inputs shared by the CUDA path, the oracle and the tests.

This package holds NONE of the method's arithmetic (no norm, attention,
projection, scheduling or metric code). It only draws random numbers and
packs them into plain arrays:

* ``shapes``  -- the model shapes of SURVEY.md section 8 (tiny, 8B, 34B, 70B/r).
* ``weights`` -- seeded random-init weights, rounded to bf16 (RNE) so both sides
  see bit-identical values.
* ``traces``  -- seeded request traces (prompt/output lengths, Poisson arrivals,
  prompt token ids) shaped like the paper's workloads (Table 4,
  P:638-651; Poisson arrivals P:669).
"""
from .shapes import ModelShape, SHAPES, get_shape  # noqa: F401
