"""Per-source-line static instruction counts inside a kernel's longest loop (nvdisasm -g of the
cubin holding it): python scripts/sass_lines.py <cubin-stem> <mangled-substring> [topN]
e.g. python scripts/sass_lines.py tab_down 'k_downILb0ELb1ELb1ELb0ELb0ELb1ELb0E' 40"""
import collections
import os
import re
import subprocess
import sys
import tempfile

LIB = "paper_1802_06130_b200/libblade_ms.so"


def main():
    stem, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(LIB)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith(stem) and f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = txt.split("\n")
    start = [i for i, l in enumerate(lines) if l.startswith(".text.") and pat in l][0]
    end = next(i for i in range(start + 1, len(lines)) if lines[i].startswith(".text.") or lines[i].startswith(".nv."))
    cur, pend, ins, lab = None, [], [], {}
    for l in lines[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"^(\.L_x_\d+):", l.strip())
        if m:
            pend.append(m.group(1))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            a = int(m.group(1), 16)
            for p in pend:
                lab[p] = a
            pend = []
            ins.append((a, m.group(2), cur))
    best = None
    for a, t, _ in ins:
        m = re.search(r"BRA.*`\((\.L_x_\d+)\)", t)
        if m and m.group(1) in lab and lab[m.group(1)] < a:
            if best is None or a - lab[m.group(1)] > best[1] - best[0]:
                best = (lab[m.group(1)], a)
    g, ops = collections.Counter(), collections.defaultdict(collections.Counter)
    for a, t, c in ins:
        if best[0] <= a <= best[1]:
            g[c] += 1
            op = t.split()
            op = op[1] if op[0].startswith("@") else op[0]
            ops[c][op.split(".")[0]] += 1
    print(f"loop {best[0]:#x}..{best[1]:#x}: {sum(g.values())} static instructions")
    for c, v in g.most_common(top):
        print(f"{v:5d} {c[0]}:{c[1]}  {dict(ops[c].most_common(5))}")


if __name__ == "__main__":
    main()
