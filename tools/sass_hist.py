#!/usr/bin/env python
"""Opcode histogram per kernel of a cubin / executable / .so (cuobjdump -sass).

    python tools/sass_hist.py <binary> [kernel-substring] [--min N]
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict


def hist(path, filt=None):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    fn, h = None, defaultdict(Counter)
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m and fn and (filt is None or filt in fn):
            ins = m.group(1).strip()
            if ins.startswith("@"):
                ins = ins.split(None, 1)[1]
            op = ins.split()[0]
            h[fn][op] += 1
    return h


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    mn = 1
    if "--min" in sys.argv:
        mn = int(sys.argv[sys.argv.index("--min") + 1])
        args = [a for a in args if a != str(mn)]
    h = hist(args[0], args[1] if len(args) > 1 else None)
    demangle = subprocess.run(["c++filt"], input="\n".join(h), capture_output=True, text=True).stdout.split("\n")
    for (fn, c), name in zip(h.items(), demangle):
        print(f"== {name}  ({sum(c.values())} instructions)")
        for op, k in c.most_common():
            if k >= mn:
                print(f"   {k:6d} {op}")


if __name__ == "__main__":
    main()
