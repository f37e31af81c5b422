"""Float64 CPU oracle for the fast CS-SAR ITA hot path (arXiv 1302.3120).

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import anything under
oracle/.  The CUDA path (paper_1302_3120_b200/) shares no code with it: no kernels,
headers, helpers, tables or constant generators.

Modules (each function cites the PAPER.md passage it follows):
  csa      CSA focusing M and approximated observation G = M^H (eq. 10-11, Theorem 1)
  rda      RDA focusing M and G = M^H with the truncated-sinc RCMC and its transpose (eq. 14-18, 23)
  ita      soft / half thresholds, k-rule and fixed-lambda rules, Algorithm 1 (eq. 7-9, 25-28)
  echo     exact periodic point-target echo (eq. 1-3) and inverse-CSA echo
  metrics  IRW / PSLR of a focused point target (P:L512 method)

Pins (tests/test_oracle_*.py, all -m "not gpu") tie every function to something other
than itself: naive-DFT dense chains, Theorem 1 adjoint identity, exact unitarity,
point-target focusing to closed-form peak / phase / resolution / PSLR, worked examples
from SPEC, brute-force scalar minimisation, the Theta = 1 one-step fixed point, fixed-
lambda objective monotonicity, and SURVEY 8(c).7 transcription anchors.

Parity unpinned: whether this CSA chain is the operator the paper intends
(PAPER.md prints no CSA phase function) — pinned only by the physics (focusing)
tests, not by paper values; the L1/2 operator constants (not printed at P:L102) — pinned
by brute-force minimisation of its defining objective.
"""
from . import csa, ita, echo, metrics, rda  # noqa: F401
