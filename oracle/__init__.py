"""fp64 CPU oracle for the hot path of arXiv:1509.03979 (Hsieh, Lu, Pei).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product (paper_1509_03979_b200/, its CUDA kernels and C ABI) never imports,
calls or links it, and this package shares no code with the product: its
transforms are scipy's DCT (and an explicit cosine matrix for tiny N), its
linear algebra is numpy.

Plain, slow, obviously correct, float64 throughout.  Every function cites the
PAPER.md line (P:n) or SPEC.md line (S:n) it follows; readings of the paper
where it is silent or garbled are listed in DESIGN.md §3 ("Readings").

Pins (tests/test_oracle_*.py, `-m "not gpu"`):
  operator      dense closed-form C_N at small N, A A^T = I, adjoint identity,
                DCT worked examples (1,1,1,1) -> (2,0,0,0) and cosine inputs.
  cg            numpy.linalg.lstsq on small supports (Thm 1-2), Thm 4 spectral
                iteration bound, Thm 5 reduced-system trace, orthogonality.
  pursuits      SPEC toy A = I_4 cases, brute-force l0 on tiny N, dense-LS
                backend equivalence, exact noiseless recovery, and hand-worked
                step pins: OMP's exclusion of S (Eq.(6)), SP's J off S and its
                RESID_ROSE halt keeping (S, x), OMPR(l, eta)'s eta swap rule
                (tests/test_oracle_pursuits.py test_*_step / *_exclude_* /
                *_resid_rose_*; each fails under a mutation of that step).
  Every step of every pursuit is pinned as above.  What no independent
                reference fixes is which support a NOISY SP run ends on at the
                configs' sizes (c2, c5): there the oracle's own full-size answer
                (tools/oracle_reference.py -> tests/golden/) is the reference,
                checked on the invariants (non-increasing residual, fixed point,
                orthogonality).
"""
from .operator import SrmOperator, DenseOperator, dct_matrix, dense_srm  # noqa: F401
from .cg import cg, reduced_cg, CgResult  # noqa: F401
from .pursuits import omp, sp, ompr, cosamp, recover, topk, PursuitResult  # noqa: F401
from .dense import brute_force_l0, lstsq_on_support  # noqa: F401
