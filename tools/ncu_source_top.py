"""Top source lines of a kernel by warp-stall samples (dev tool).

ncu -i REP --page source --csv --print-source cuda,sass --kernel-name regex:K --launch-count 1 > SRC.csv
python tools/ncu_source_top.py SRC.csv [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = []
    hdr = None
    fname = ""
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
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    v = int(r[i])
                except ValueError:
                    continue
                if v:
                    stalls[h[6:]] = v
        out.append((samples, fname, r[0], r[1].strip()[:90], stalls))
    tot = sum(o[0] for o in out) or 1
    print("total samples", tot)
    for s, f, ln, src, st in sorted(out, reverse=True)[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100.0 * s / tot:5.1f}% {f}:{ln:>5} {src:<90} {top3}")


if __name__ == "__main__":
    main()
