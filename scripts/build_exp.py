"""Build A/B variants of libblade_ms.so into exp/ (git-ignored .so files that still travel to the
GPU box): python scripts/build_exp.py name -DFLAG=V ... ; run with BLADE_MS_LIB=exp/name.so."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1802_06130_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = Path(__file__).resolve().parents[1] / "exp" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
b.build(force=True, extra=flags, out=out)
print(out)
