"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
per CUDA source line and per enclosing function.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict

FUNC = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__)[^;{]*?\b([A-Za-z_]\w*)\s*\(")


def enclosing_functions(path):
    """line -> name of the most recent __device__/__global__ definition."""
    names, cur = {}, "?"
    try:
        lines = open(path).read().split("\n")
    except OSError:
        return names
    for i, ln in enumerate(lines, 1):
        m = FUNC.match(ln.strip())
        if m:
            cur = m.group(1)
        names[i] = cur
    return names


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    reasons = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_no_inst", "stall_branch_resolving", "stall_selected"]
    per_line = defaultdict(lambda: [0] * (3 + len(reasons)))
    per_func = defaultdict(lambda: [0] * (3 + len(reasons)))
    fname, hdr, funcs = None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1]
            funcs = enclosing_functions(fname)
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name",) or not r[0].isdigit():
            continue
        if r[2] != "-":  # sass row, counted through its source line
            continue
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            nis = int(r[hdr.index("Warp Stall Sampling (Not-issued Samples)")])
            ins = int(r[hdr.index("Instructions Executed")])
            rs = [int(r[hdr.index(x)]) for x in reasons]
        except (ValueError, IndexError):
            continue
        ln = int(r[0])
        key = (fname.split("/")[-1], ln, r[1].strip()[:70])
        for acc in (per_line[key], per_func[(fname.split("/")[-1], funcs.get(ln, "?"))]):
            acc[0] += samp
            acc[1] += nis
            acc[2] += ins
            for j, x in enumerate(rs):
                acc[3 + j] += x
    tot = sum(v[0] for v in per_func.values()) or 1
    toti = sum(v[2] for v in per_func.values()) or 1
    short = ["wait", "short", "long", "noins", "branch", "sel"]
    print(f"{'function':40s} {'stall%':>7s} {'inst%':>7s} " + " ".join(f"{x:>6s}" for x in short) + "  (% of all samples)")
    for k, v in sorted(per_func.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0][:16] + ':' + k[1]:40s} {100 * v[0] / tot:7.2f} {100 * v[2] / toti:7.2f} "
              + " ".join(f"{100 * x / tot:6.2f}" for x in v[3:]))
    print()
    for k, v in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0][:14]}:{k[1]:<5d} {100 * v[0] / tot:6.2f} {100 * v[2] / toti:6.2f} "
              + " ".join(f"{100 * x / tot:5.2f}" for x in v[3:7]) + f"  {k[2]}")


if __name__ == "__main__":
    main()
