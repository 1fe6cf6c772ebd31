"""Randomised parity sweep on one GPU: random shapes, pyramid depths, footprints, bucket layouts,
windows and batch sizes through the C ABI against the fp64 oracle with the GPU suite's rule
(tests/test_gpu_parity._full_parity). A measurement / hardening aid: prints one line per case
and a summary; failures are listed with their seed so they can be turned into a test.

    python scripts/fuzz_parity.py [cases] [seed] [identity|ycc|xband] [big]

`identity` (optionally with `ycc`: per-channel banks) runs the bit-identity properties instead (per-frame calls, row bands, chunked schedule,
host-buffer call against blade_ms_denoise; no oracle).
"""
import sys
import traceback
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


from tests.fuzz_cases import draw, run_case, run_identity_case, run_xband_case, run_ycc_case  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ident = "identity" in sys.argv[3:]
    rng = np.random.default_rng(seed0)
    fails = []
    for i in range(cases):
        p = draw(rng, big="big" in sys.argv[3:])
        seed = seed0 * 1000 + i
        try:
            worst = 0.0
            if ident:
                run_identity_case(p, seed, channels=3 if "ycc" in sys.argv[3:] else 1)
            elif "xband" in sys.argv[3:]:
                ran = run_xband_case(p, seed, channels=3 if "ycc" in sys.argv[3:] else 1)
                worst = 0.0 if ran else float("nan")  # nan: the layout refused the split
            elif "ycc" in sys.argv[3:]:
                run_ycc_case(p, seed)
            else:
                worst = run_case(p, seed)
            print(f"ok   seed={seed} {p} max|gpu-oracle|={worst:.2e}", flush=True)
        except Exception as e:  # noqa: BLE001 (report and continue)
            fails.append((seed, p, repr(e)[:300]))
            print(f"FAIL seed={seed} {p}: {e!r}"[:600], flush=True)
            traceback.print_exc(limit=3)
    print(f"{cases - len(fails)}/{cases} cases within the parity rule; failures: {fails}")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
