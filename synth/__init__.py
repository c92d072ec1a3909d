"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no simplification, no search,
no cost evaluation): it only builds decomposed graphs (DG: conflict edges CE
and stitch edges SE over vertex/segment ids, §2.1 "E = {CE ∪ SE}")
in CSR form, shaped like the layout graphs the paper decomposes (Table 1).
"""
from .graph import DecompGraph, from_edges, concat, split, upper_csr, stitch_pairs
from .layouts import (TABLE1, make_layout, iscas_layout, config_graphs,
                      stress_components, fixtures)

__all__ = ["DecompGraph", "from_edges", "concat", "split", "upper_csr", "stitch_pairs", "TABLE1", "make_layout",
           "iscas_layout", "config_graphs", "stress_components", "fixtures"]
