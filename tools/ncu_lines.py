"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source sass,cuda` (dev tool).

python tools/ncu_lines.py report.ncu-rep KERNEL_REGEX [N]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
    fname, hdr = "", None
    by_line = collections.Counter()
    stalls = collections.defaultdict(collections.Counter)
    text = {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        key = (fname, int(r[0]) if r[0].isdigit() else -1)
        def num(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        s = num(r[4])
        by_line[key] += s
        text.setdefault(key, r[1].strip()[:90])
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                stalls[key][h[6:]] += num(r[i])
    tot = sum(by_line.values()) or 1
    for key, s in by_line.most_common(top):
        st = ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in stalls[key].most_common(2) if s)
        print(f"{100 * s / tot:5.1f}%  {key[0]}:{key[1]:<5} {text[key]:<90} [{st}]")


if __name__ == "__main__":
    main()
