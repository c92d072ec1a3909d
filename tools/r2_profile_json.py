"""profiles/r2_kernels*.json from an ncu --set full report plus the node counts
of the profiled call (dev tool).

python tools/r2_profile_json.py REPORT.ncu-rep OUT.json "source" [PROFILE_RUN_JSON]

PROFILE_RUN_JSON: the line bench.py --profile-launches printed (last_call_nodes,
last_call_heavy_nodes): the warp instructions per search node of the light and
heavy kernels are inst_executed / nodes (the roofline denominator of the search
kernels).
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
    subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), rep, out, src], check=True)
    d = json.load(open(out))
    if len(sys.argv) > 4:
        run = json.loads(open(sys.argv[4]).read().strip().splitlines()[-1])
        tot, heavy = run.get("last_call_nodes"), run.get("last_call_heavy_nodes")
        if tot:
            light = tot - heavy
            k = d["kernels"]
            if "mpld_exact_cover_search" in k and light:
                k["mpld_exact_cover_search"]["nodes"] = light
                k["mpld_exact_cover_search"]["inst_per_node"] = k["mpld_exact_cover_search"]["inst_executed"] / light
            if "mpld_exact_cover_search_heavy" in k and heavy:
                k["mpld_exact_cover_search_heavy"]["nodes"] = heavy
                k["mpld_exact_cover_search_heavy"]["inst_per_node"] = (
                    k["mpld_exact_cover_search_heavy"]["inst_executed"] / heavy)
            d["profiled_call_nodes"] = {"total": tot, "heavy": heavy}
    json.dump(d, open(out, "w"), indent=1)
    for name, v in d["kernels"].items():
        if "inst_per_node" in v:
            print(name, "inst/node", round(v["inst_per_node"], 1))


if __name__ == "__main__":
    main()
