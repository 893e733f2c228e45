"""The drop-in surface: every name the reference package exports resolves
(tests/golden/reference_exports.json, from pkg/src/jhsvd/__init__.py:10-81)
except the documented exclusions, and the robust-norm / rotation API gives
the reference's values (tests/golden/api.npz, make_api_golden.py)."""

import json
import math

import numpy as np
import pytest

import paper_1401_2720_b200 as J
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def api():
    return np.load(GOLDEN / "api.npz")


def test_every_reference_export_resolves():
    names = json.loads((GOLDEN / "reference_exports.json").read_text())["names"]
    missing = [n for n in names if not hasattr(J, n)]
    assert sorted(missing) == sorted(J.REFERENCE_EXCLUSIONS)
    assert len(names) > 50


def test_column_mapping_carries_fast_exchanges():
    m = J.optimize_mapping(J.make_strategy("rrow", 8), J.Topology(4))
    assert m.fast_exchanges == 3  # reference test_distsim.py:48-50
    m2 = J.ColumnMapping(m.g, m.assignments, m.moves, m.fast_exchanges)
    assert m2 == m
    u = J.legal_mapping(J.make_strategy("rrow", 8))
    assert u.fast_exchanges == 7  # NVSwitch: every transition is fast


def test_scalar_helpers_match_reference(api):
    for f, t, up, want in api["scale_exp"]:
        assert J.scale_exponent(f, t, "up" if up else "down") == int(want)
    for e, v, je, ve in api["common_form"]:
        r = J.common_form(J.ScaledSquare(int(e), v))
        assert (r.scale_exp, r.value) == (int(je), ve)
    for ja, va, jb, vb, jr, vr in api["add_scaled"]:
        r = J.add_scaled(J.ScaledSquare(int(ja), va), J.ScaledSquare(int(jb), vb))
        assert (r.scale_exp, r.value) == (int(jr), vr)
    with pytest.raises(ValueError):
        J.scale_exponent(0.0, 1.0, "up")
    with pytest.raises(ValueError):
        J.common_form(J.ScaledSquare(0, -1.0))


def test_safe_bounds_rejects_empty():
    with pytest.raises(ValueError):
        J.safe_bounds(0)


@pytest.mark.gpu
def test_sum_squares_and_norm2_bitwise(api):
    k = 0
    while f"ss{k}_in" in api.files:
        x = api[f"ss{k}_in"]
        chunk, force = (int(v) for v in api[f"ss{k}_opt"])
        ss = J.sum_squares(x, chunk=chunk, force_scaled=bool(force))
        assert ss.scale_exp == int(api[f"ss{k}_sqj"][0]), k
        assert ss.value == api[f"ss{k}_sq"][1], k
        js, s = J.norm2(x, chunk=chunk, force_scaled=bool(force))
        assert (js, s) == (int(api[f"ss{k}_normj"][0]), api[f"ss{k}_norm"][0]), k
        k += 1
    assert k == 42
    assert J.norm2_value(np.array([3.0, 4.0])) == 5.0
    with pytest.raises(ValueError):
        J.norm2(np.array([1.0, math.inf]))


@pytest.mark.gpu
def test_compute_rotation_bitwise(api):
    for (hpp, hqq, hpq, t), (cs, tn, ok, proper) in zip(api["rot_in"], api["rot_out"]):
        kind = "trig" if t > 0 else "hyp"
        if not ok:
            with pytest.raises(J.HyperbolicDomainError):
                J.compute_rotation(J.PivotGram(hpp, hqq, hpq), kind)
            continue
        p = J.compute_rotation(J.PivotGram(hpp, hqq, hpq), kind)
        assert (p.cs, p.tn, p.proper) == (cs, tn, bool(proper)), (hpp, hqq, hpq, kind)
    cs, tn, ok = J.compute_rotations(api["rot_in"][:, :3], api["rot_in"][:, 3])
    assert np.array_equal(ok, api["rot_out"][:, 2] != 0)
