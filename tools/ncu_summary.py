"""Summarise an `ncu --set full` report into profiles/<round>_kernels.json (dev tool).

python tools/ncu_summary.py REPORT.ncu-rep OUT.json "source description"
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    def f(d, name):
        try:
            return float(d[col[name]].replace(",", ""))
        except (KeyError, ValueError):
            return None

    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def nbytes(d, name):
        v = f(d, name)
        return 0.0 if v is None else v * scale.get(units[col[name]], 1.0)

    kernels = {}
    for d in data:
        full = d[col["Kernel Name"]].split("(")[0]
        name = full.split("::")[-1].split("<")[0].strip()
        if "<" in full and ("unsigned long long" in full or full.rstrip().endswith("unsigned int>")):
            name += "<64>" if "unsigned long long" in full else "<32>"  # word class of the heavy search
        if name in kernels and not ("--all" in sys.argv):  # a later launch of the same kernel: keep the first
            continue
        if name in kernels:
            name += "#%d" % sum(1 for x in kernels if x.split("#")[0] == name)
        stalls = {}
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(d[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
        kernels[name] = {
            "duration_us": f(d, "gpu__time_duration.sum"),
            "dram_bytes": nbytes(d, "dram__bytes_read.sum") + nbytes(d, "dram__bytes_write.sum"),
            "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_hit_pct": f(d, "lts__t_sector_hit_rate.pct"),
            "inst_executed": f(d, "smsp__inst_executed.sum"),
            "grid": int(f(d, "launch__grid_size") or 0),
            "block": int(f(d, "launch__block_size") or 0),
            "regs": int(f(d, "launch__registers_per_thread") or 0),
            "stall_top_pct": {k: round(100 * v / tot, 1) for k, v in top},
            # the counters the north_star names: divergence (active threads per executed
            # warp instruction, 32 = none), issue-slot use, L2 / L1+shared throughput
            "threads_per_inst": f(d, "smsp__thread_inst_executed_per_inst_executed.ratio"),
            "divergent_branch_targets": f(d, "smsp__sass_branch_targets_threads_divergent.sum"),
            "issue_active_pct": f(d, "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "l2_throughput_pct": f(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l1tex_throughput_pct": f(d, "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "shared_wavefronts_pct": f(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "dram_throughput_pct": f(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        }
    json.dump({"source": src, "kernels": kernels}, open(out, "w"), indent=1)
    for k, v in kernels.items():
        print(k, round(v["duration_us"], 1), "us", round(v["dram_bytes"] / 1e6, 2), "MB", v["stall_top_pct"],
              "thr/inst", v["threads_per_inst"], "issue%", v["issue_active_pct"], "L2%", v["l2_throughput_pct"],
              "L1%", v["l1tex_throughput_pct"], "shm%", v["shared_wavefronts_pct"], "warps%", v["warps_active_pct"])


if __name__ == "__main__":
    main()
