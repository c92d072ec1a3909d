"""CPU oracle for the MPLD hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain, slow, obviously-correct Python written from PAPER.md (arxiv 2303.14335),
following the paper's order and notation; every function cites the passage it
implements.  Readings of silent / ambiguous passages are listed in DESIGN.md §2.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this package.  The CUDA path under
`paper_2303_14335_b200/` shares no code with it and never imports it.

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): brute-force k^n enumeration
of Eq. 1 on tiny graphs, closed forms (K_n optimum = Turán deficit, odd/even
cycles, K_{k+1}), Fig. 1 (4-clique not 3-colourable; two stitches
remove the conflict), a pruning-free enumeration of the canonical search tree
(colours, not just cost), DLX cover/uncover round trips (Eq. 2), and the
recovery/simplification invariants.  Every function is pinned; none is
"parity unpinned".
"""
from .mpld import (W_CONF, alpha_units, validate, simplify, lowbias32, components,
                   recover, evaluate, solve_component, decompose)
from .dlx import DLXMatrix, algorithm_x

__all__ = ["W_CONF", "alpha_units", "validate", "simplify", "lowbias32", "components",
           "recover", "evaluate", "solve_component", "decompose", "DLXMatrix", "algorithm_x"]
