"""FireQ W4A8-FP linear-layer oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, fp64 where the
arithmetic is not fixed by the method) of what the hot path computes, written
from arXiv 2505.20839 (``P:NNN`` = /root/reference/PAPER.md line) and the
readings fixed in DESIGN.md / SURVEY.md section 8(c).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import anything from here.
The product path (``paper_2505_20839_b200``) never imports this package and
shares no code with it: no kernels, headers, tables or constant generators.

Modules
  numerics  E4M3 ("fn") and BF16 codecs, RN / RZ rounding
  layout    packed-INT4 / scale byte index formula (layout version 1)
  quant     CAS, PTS, INT4 group quantization
            (P:45-48), FP8 activation quantization
  gemm      16-entry LUT, fp64 reference GEMM (P:61-65, P:129-130,
            P:175), the G4 tolerance criterion

Parity pins: every function is pinned in tests/test_oracle_*.py against
something other than itself (exact-rational brute force, library casts,
closed forms, the paper's constants, golden fixtures).  Functions with no
such pin are listed as "parity unpinned" below and in DESIGN.md:

  parity unpinned: none of the encodings; the GEMM is pinned only up to
  fp64 rounding order (a library matmul serves as the contraction step).
"""
