# round 2: tile pipeline on the GPU (dev tool)
mkdir -p gpurun_out
python - > gpurun_out/gates.log 2>&1 <<'PY'
import sys, torch; sys.path.insert(0, ".")
import bench, paper_2303_14335_b200 as mp
dev = torch.device("cuda:0"); torch.cuda.set_device(0); s = torch.cuda.current_stream()
for cfg in (1, 3):
    it = bench.workload_items(cfg, 0, bench.default_replicas(cfg))[0]
    d = bench.DeviceItem(it, dev); ctx = mp.Context(0, it.g.n, it.g.n_layouts)
    gates = []
    for i in range(20):
        d.run(ctx, s, mp.MPLD_FLAG_VALIDATE); torch.cuda.synchronize(); gates.append(int(ctx.debug()[88]))
    gates2 = []
    for i in range(10):
        d.run(ctx, s, 0); torch.cuda.synchronize(); gates2.append(int(ctx.debug()[88]))
    print(cfg, "validate", gates, "novalidate", gates2, flush=True)
PY
cat gpurun_out/gates.log | tail -5
timeout 600 python tools/tile_probe.py 1 2 3 > gpurun_out/tile_probe.log 2>&1; echo "probe rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/tile_probe.log"):
    if not l.startswith("{"):
        print(l.rstrip()[:300]); continue
    d = json.loads(l)
    print(d["config"], d["item"], "gate", d["gate"], "same", d["same_colors_counts_cost_stats"], "whole", d["whole_ms"], "tile", d["tile_ms"])
    print("   tile us", d["tile_kernels_us"])
PY
timeout 900 python -m pytest tests/test_gpu_tiles.py -q -x > gpurun_out/t_tiles.log 2>&1; echo "tiles rc=$?"; tail -25 gpurun_out/t_tiles.log
