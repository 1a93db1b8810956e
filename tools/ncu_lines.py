"""Attributes an ncu source-page export (SASS, per-instruction samples) to CUDA source lines
using the -lineinfo tables of the cubin:

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all build/cand_v0s.cu.o ; nvdisasm -g -c cand_v0s.sm_100a.cubin > all.sass
    python tools/ncu_lines.py sass.csv all.sass <mangled kernel name> [top]
"""
import collections
import csv
import re
import sys


def line_map(sass_path, fn):
    """offset -> (file, line) for function fn from `nvdisasm -g -c` output."""
    out, cur, inside = {}, None, False
    for ln in open(sass_path):
        if ln.startswith(".text." + fn + ":") or ln.startswith(fn + ":"):
            inside = True
            continue
        if inside and ln.startswith("//----") and fn not in ln:
            break
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            f, l = m.group(1).split("/")[-1], int(m.group(2))
            if f.endswith((".cuh", ".cu")) or cur is None:
                cur = (f, l)
            # a CUDA library helper (min, max, intrinsics) is charged to the preceding line of ours
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out.setdefault(int(m.group(1), 16), cur)
    return out


def main():
    sass_csv, sass_txt, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    data = rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    base = int(data[0][0], 16)
    lm = line_map(sass_txt, fn)
    S = "Warp Stall Sampling (All Samples)"
    E = "Instructions Executed"
    samp, inst = collections.Counter(), collections.Counter()
    for r in data:
        off = int(r[0], 16) - base
        key = lm.get(off, ("?", 0))
        samp[key] += int(r[ix[S]] or 0)
        inst[key] += int(r[ix[E]] or 0)
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"{'samples':>8} {'instr':>8}  line")
    for key, s in samp.most_common(top):
        print(f"{100 * s / ts:7.2f}% {100 * inst[key] / ti:7.2f}%  {key[0]}:{key[1]}")


if __name__ == "__main__":
    main()
