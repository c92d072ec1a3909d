"""The graph build of the upper-triangle upload alone, a few submits (dev tool; run under ncu -k regex:graph_build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_14335_b200 as mp  # noqa: E402
import synth  # noqa: E402

graphs = []
for r in range(16):
    gs, k, alpha = synth.config_graphs(1, seed=10 * r)
    graphs += gs
b = synth.concat(graphs)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
ud, uc = synth.upper_csr(b)
ud, uc, pairs, lo = pin(ud), pin(uc), pin(synth.stitch_pairs(b)), pin(b.layout_offsets)
ctx = mp.Context(0, b.n, b.n_layouts)
for i in range(4):
    r = ctx.wait(ctx.submit_upper(lo, b.n, ud, uc, pairs, k, alpha, 0, 1))
print("ok", r["stats"]["error"])
