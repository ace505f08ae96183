"""Trace CSV and placement JSON in the reference's formats, pinned against
files the reference itself wrote (tests/golden/make_formats.py)."""

from pathlib import Path

import numpy as np
import pytest

import paper_2508_09591_b200 as hm

GOLD = Path(__file__).resolve().parent / "golden"


def test_trace_roundtrip_bytes(tmp_path):
    entries = hm.load_trace(GOLD / "trace_ref.csv", 16)
    assert [(i, l) for i, l, _ in entries] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert all(m.bits.shape == (64, 16) and m.top_k == 2 for _, _, m in entries)
    out = tmp_path / "t.csv"
    hm.save_trace(entries, out)
    assert out.read_bytes() == (GOLD / "trace_ref.csv").read_bytes()


def test_trace_matches_reference_generator():
    # the masks in the golden trace are the reference generator's output for
    # these seeds; our host generator (same PCG64 stream) reproduces them
    entries = hm.load_trace(GOLD / "trace_ref.csv", 16)
    for it, layer, m in entries:
        seed = hm.layer_seed(5, it, layer)
        want = (hm.generate_uniform(64, 16, 2, seed) if layer == 0
                else hm.generate_skewed(64, 16, 2, 1.2, seed))
        assert np.array_equal(m.bits, want.bits)


def test_placement_roundtrip_bytes(tmp_path):
    pl = hm.load_placements(GOLD / "placement_ref.json", 16)
    assert sorted(pl) == [0, 1]
    assert list(pl[0].slot_to_expert[[3, 12]]) == [12, 3]
    out = tmp_path / "p.json"
    hm.save_placements(pl, 16, out)
    assert out.read_bytes() == (GOLD / "placement_ref.json").read_bytes()
    with pytest.raises(ValueError):
        hm.load_placements(GOLD / "placement_ref.json", 32)


def test_trace_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("iter,layer,token,experts\n0,0,0,1;1\n")
    with pytest.raises(hm.TraceFormatError):
        hm.load_trace(bad, 16)
    bad.write_text("iter,layer,tok,experts\n")
    with pytest.raises(hm.TraceFormatError):
        hm.load_trace(bad, 16)


def test_runtime_params_packaged_and_loaded():
    """The B200 alpha/beta of the runtime [P, L] transports ship in the
    reference's params schema (tools/calibrate.py --runtime) and load into
    the transport choice; a flat hierarchy uses the 'std' entry only."""
    import json
    from paper_2508_09591_b200.topology import load_params
    from paper_2508_09591_b200.transport import PARAMS_DIR, default_params, runtime_topology
    files = sorted(PARAMS_DIR.glob("b200_runtime_n*.json"))
    assert [f.name for f in files] == ["b200_runtime_n2.json", "b200_runtime_n4.json"]
    for f in files:
        raw = json.loads(f.read_text())
        assert set(raw) == {"std", "inter.1", "intra.1"}
        p = load_params(f, 2)
        assert p.alpha_std == raw["std"]["alpha"] and p.inter(1)[1] == raw["inter.1"]["beta"]
    assert runtime_topology(8, 2, 128, 2048).level_fanouts == (2, 4)
    assert runtime_topology(8, 4, 128, 2048).level_fanouts == (4, 2)
    assert runtime_topology(8, 1, 128, 2048).level_fanouts == (8,)
    assert runtime_topology(8, 8, 128, 2048).level_fanouts == (8,)
    p2 = default_params(2, 2)
    assert p2 == load_params(PARAMS_DIR / "b200_runtime_n2.json")
    flat = default_params(8, 1)          # N = 8: nearest fit (n4), std entry only
    n4 = load_params(PARAMS_DIR / "b200_runtime_n4.json")
    assert flat.num_levels == 1 and flat.alpha_std == n4.alpha_std and flat.beta_std == n4.beta_std
