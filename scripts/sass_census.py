"""Instruction census of the built library (cuobjdump -sass): per kernel, the counts of the
mnemonics that show which units it uses (TMA: UTMALDG / UBLKCP; tensor cores: DMMA; packed fp32:
FFMA2 / FADD2 / FMUL2; CUDA-core FFMA / DFMA; shared-memory LDS widths; SHFL). Static counts
(instructions in the binary, not executed).   python scripts/sass_census.py [lib.so]"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

lib = sys.argv[1] if len(sys.argv) > 1 else str(Path(__file__).resolve().parents[1] / "paper_1802_06130_b200" / "libblade_ms.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UTMALDG", "UBLKCP", "DMMA", "HMMA", "FFMA2", "FADD2", "FMUL2", "FFMA", "DFMA", "LDS.128", "LDS.64", "LDS",
        "SHFL", "LDGSTS", "SYNCS"]
cur, counts, order = None, {}, []
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        if cur not in counts:
            counts[cur] = Counter()
            order.append(cur)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if cur and m:
        op = m.group(1)
        base = op.split(".")[0]
        for k in keys:
            if op == k or op.startswith(k + ".") and k in ("LDS.128", "LDS.64") or base == k and "." not in k:
                counts[cur][k] += 1
                break


def short(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()[:110]
    except OSError:
        return name[:110]


want = re.compile(r"k_stage_tma|k_stage_ph|k_down|k_train_gram|k_stage_fixup")
print("static SASS counts per kernel (" + Path(lib).name + ")")
print("kernel".ljust(112) + " ".join(k.rjust(8) for k in keys))
seen = set()
for f in order:
    s = short(f)
    if not want.search(s) or s in seen:
        continue
    seen.add(s)
    print(s.ljust(112) + " ".join(str(counts[f][k]).rjust(8) for k in keys))
