"""Static instruction mix of a kernel's hottest loop (the span of its longest backward branch)
from `cuobjdump -sass` of the built library: python scripts/sass_loop.py <mangled-name-substring>
[--skip lo:hi ...]. Used to count per-pixel instructions of issue-bound kernels before a GPU run."""
import collections
import re
import subprocess
import sys

LIB = "paper_1802_06130_b200/libblade_ms.so"


def main():
    pat = sys.argv[1]
    skips = [tuple(int(x, 16) for x in s.split(":")) for s in sys.argv[2:] if ":" in s]
    names = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    fns = sorted(set(re.findall(r"Function : (\S+)", names)))
    fn = [f for f in fns if pat in f]
    assert len(fn) >= 1, f"no kernel matching {pat}"
    fn = fn[0]
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True).stdout
    ins = []
    for line in out.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and (best is None or a - tgt > best[1] - best[0]):
                best = (tgt, a)
    c = collections.Counter()
    for a, t in ins:
        if best[0] <= a <= best[1] and not any(lo <= a < hi for lo, hi in skips):
            op = t.split()
            op = op[1] if op[0].startswith("@") else op[0]
            c[op.split(".")[0]] += 1
    print(fn)
    print(f"loop {best[0]:#x}..{best[1]:#x}: {sum(c.values())} instructions")
    print(" ".join(f"{k}:{v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
