"""CPU oracle for the cDMD hot path (arXiv 1512.04205) — TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, fp64 NumPy implementation of what the hot path
computes, written step by step from PAPER.md (Algorithm 1; Remark 3,
P:363-369; Eq. thres) and from the measurement-matrix definitions
of DESIGN.md §3 (our reading of P:374-394).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package ``paper_1512_04205_b200`` never imports it, shares no code with it,
and fails loudly when its CUDA library is missing.

Parity status of each function is stated in its module header; every function
here is pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``.
"""

from . import philox, sensing, cdmd  # noqa: F401
