"""Oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU (numpy/scipy, float64/complex128)
implementation of what the hot path computes, written from PAPER.md
(/root/reference/PAPER.md; cited as P:line) and SURVEY.md App. A.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package. The CUDA product path shares no
code with it and never imports it. Inputs come from the separate `synth`
module, which holds none of the method's arithmetic.
"""
from .linalg import Breakdown, gram, thin_qr, small_solve, unitary_qr_stack  # noqa: F401
from .solvers import METHODS, SOLVERS, Result, solve  # noqa: F401
