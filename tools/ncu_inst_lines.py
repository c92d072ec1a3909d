"""Warp instructions per source line of one kernel (dev tool), optionally per
search iteration.

ncu -i REP --page source --csv --print-source cuda,sass --launch-count 1 > SRC.csv
python tools/ncu_inst_lines.py SRC.csv [ITERATIONS] [N]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    iters = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    hdr, fname, out = None, "", collections.Counter()
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0]:
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        out[(fname, int(r[0]), r[1].strip()[:96])] += ie
    tot = sum(out.values())
    print(f"warp instructions {tot:.0f}; per iteration ({iters:.0f} iterations) {tot / iters:.1f}")
    for (f, ln, src), v in sorted(out.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v / iters:9.1f} {100 * v / tot:5.1f}% {f}:{ln} {src}")


if __name__ == "__main__":
    main()
