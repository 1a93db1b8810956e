"""Per-source-line (and per-function-region) totals of an ncu source-page SASS export:
instructions executed, stall samples, shared-memory wavefronts (+ excessive), global
sectors.  Usage:

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all build/cand_v0s.cu.o ; nvdisasm -g -c cand_v0s.sm_100a.cubin > all.sass
    python tools/ncu_regions.py sass.csv all.sass <mangled kernel> [top]
"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines  # noqa: E402

COLS = ["Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Excessive", "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Excessive"]


def main():
    sass_csv, sass_txt, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
    rows = list(csv.reader(open(sass_csv)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    base = int(data[0][0], 16)
    lm = ncu_lines.line_map(sass_txt, fn)
    acc = collections.defaultdict(lambda: [0] * len(COLS))
    ops = collections.defaultdict(collections.Counter)
    for r in data:
        key = lm.get(int(r[0], 16) - base, ("?", 0))
        for k, c in enumerate(COLS):
            v = r[ix[c]]
            acc[key][k] += int(float(v)) if v not in ("", None) else 0
        op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        ops[key][op.split(".")[0]] += int(float(r[ix["Instructions Executed"]] or 0))
    tot = [sum(a[k] for a in acc.values()) or 1 for k in range(len(COLS))]
    print("totals: " + "  ".join(f"{c}={t:.4g}" for c, t in zip(COLS, tot)))
    print(f"{'inst%':>7} {'stall%':>7} {'shWF%':>7} {'shExc%':>7} {'glSec%':>7}  line  top-ops")
    for key, a in sorted(acc.items(), key=lambda kv: -kv[1][1])[:top]:
        top_ops = ",".join(f"{o}:{100 * n / max(1, a[0]):.0f}" for o, n in ops[key].most_common(4))
        print(f"{100 * a[0] / tot[0]:7.2f} {100 * a[1] / tot[1]:7.2f} {100 * a[2] / tot[2]:7.2f} "
              f"{100 * a[3] / tot[3]:7.2f} {100 * a[4] / tot[4]:7.2f}  {key[0]}:{key[1]}  {top_ops}")


if __name__ == "__main__":
    main()
