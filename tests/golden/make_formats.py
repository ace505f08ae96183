"""Golden trace CSV / placement JSON written by the REFERENCE (build container
only; reads /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_formats.py

Outputs: tests/golden/trace_ref.csv (routing.py:218-227 save_trace of four
seeded masks) and tests/golden/placement_ref.json (cli.py:193-198
_save_placements of two layers' placements after a planned swap).
"""

import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import hiera2a as H  # noqa: E402
from hiera2a import cli as HC  # noqa: E402
from hiera2a import routing as HR  # noqa: E402

OUT = Path(__file__).resolve().parent


def masks():
    out = []
    for it in range(2):
        for layer in range(2):
            seed = H.layer_seed(5, it, layer)
            m = (HR.generate_uniform(64, 16, 2, seed) if layer == 0
                 else HR.generate_skewed(64, 16, 2, 1.2, seed))
            out.append((it, layer, m))
    return out


def main():
    HR.save_trace(masks(), OUT / "trace_ref.csv")
    p0 = HR.Placement.identity(16).swapped(3, 12)
    p1 = HR.Placement.identity(16).swapped(0, 15).swapped(5, 9)
    HC._save_placements({0: p0, 1: p1}, 16, OUT / "placement_ref.json")


if __name__ == "__main__":
    main()
