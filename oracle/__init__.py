"""CPU oracle for arXiv 1703.09085 (accumulated-update H-matrix arithmetic).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
from this package.  The product path (`paper_1703_09085_b200`) never
imports, calls or links it, and this package never imports the product
path; the two share no code.  The only shared module is `hm_inputs`
(geometry + probe vectors, no method arithmetic).

Plain, slow, obviously-correct Python 3 + NumPy/SciPy in FP64.  Each
function cites the PAPER.md passage it follows ("P:L<line>", with the
section / figure).  Readings of ambiguous passages are those of
SURVEY.md §8(c) and are listed in DESIGN.md §3.

Modules
  kernel    BEM-like kernel matrix entries (BASELINE.json configs)
  trees     cluster tree / block tree (Defs 2.1-2.2)
  lowrank   TRUNC_eps, rkadd, rowmerge, rkmerge (Figs 2, 4)
  hmatrix   H-matrix container, build, addeval/addevaltrans, rkupdate
            (Def 2.4, Figs 1, 3)
  product   product tree; standard (S0), literal accumulated (S1) and
            level-batched accumulated (S2) multiplication (§4, Figs 5-7)
  factor    H-LR / H-Cholesky with accumulators (§6)

Parity status of each function is stated in its docstring; functions with
no independent pin say "parity unpinned" (also listed in DESIGN.md).
"""
