"""configs[2] heavy-search time against the greedy starting incumbent (dev tool):
MPLD_GREEDY_SALT / MPLD_GREEDY_ROUNDS are read at context creation.

python tools/greedy_sweep.py SALT ROUNDS [CONFIG] [FLAGS]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MPLD_GREEDY_SALT"] = sys.argv[1]
os.environ["MPLD_GREEDY_ROUNDS"] = sys.argv[2]
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
extra = int(sys.argv[4]) if len(sys.argv) > 4 else 0

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_14335_b200 as mp  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
it = bench.workload_items(cfg, 0, bench.default_replicas(cfg))[0]
d = bench.DeviceItem(it, dev)
ctx = mp.Context(0, it.g.n, it.g.n_layouts)
for _ in range(2):
    d.run(ctx, s, mp.MPLD_FLAG_VALIDATE | extra)
torch.cuda.synchronize()
ctx.reset_timing()
ctx.set_timing(True)
for _ in range(5):
    d.run(ctx, s, mp.MPLD_FLAG_VALIDATE | extra)
torch.cuda.synchronize()
kt = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.kernel_times().items() if v[1]}
st = d.stats_dict()
dbg = ctx.debug()
print(json.dumps({"flags": extra, "heavy_comps": int(dbg[93]), "heavy_nodes": int(dbg[85]), "salt": sys.argv[1], "rounds": sys.argv[2], "heavy_us": kt.get("mpld_exact_cover_search_heavy"),
                  "steps": st["steps"], "kernels": kt}))
