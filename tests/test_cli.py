"""CLI, file formats and test generation against the reference's own
outputs (tests/golden/cli/, written by tests/golden/make_cli_golden.py from
the reference jhsvd.cli).  CPU tests cover the host paths (strategy tables,
testgen files, JHSV / CSV round trips, error handling); GPU tests the solver
reports, the device file streaming and the GPU test generator."""

import contextlib
import io
import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_1401_2720_b200 import cli, matio
from paper_1401_2720_b200.blockkernel import Signature
from paper_1401_2720_b200.testgen import SpectrumSpec, gen_factor, gen_spectrum

GOLD = Path(__file__).resolve().parent / "golden" / "cli"


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def strip_wall(text):
    rep = json.loads(text)
    rep.pop("wall_time_s", None)
    rep["config"]["input"] = "<input>"
    return json.dumps(rep, indent=2) + "\n"


@pytest.mark.parametrize("kind,n,expand", [("rrow", 16, 1), ("mm", 32, 0), ("rcol", 8, 2),
                                           ("bl", 12, 0)])
def test_strategy_gen_matches_reference(kind, n, expand):
    rc, text = run(["strategy", "gen", "--kind", kind, "--n", str(n), "--expand", str(expand)])
    assert rc == 0
    assert text == (GOLD / f"strategy_{kind}_{n}_x{expand}.txt").read_text()


def test_strategy_gen_usage_error():
    assert run(["strategy", "gen", "--kind", "mm", "--n", "8", "--expand", "1"])[0] == 2


@pytest.mark.parametrize("typ,n,seed", [(3, 64, 5), (2, 48, 9)])
def test_testgen_files_bitwise(typ, n, seed, tmp_path):
    stem = f"tg_t{typ}_n{n}_s{seed}"
    out, lam = tmp_path / "g.jhsv", tmp_path / "l.csv"
    rc, _ = run(["testgen", "--type", str(typ), "--n", str(n), "--seed", str(seed),
                 "--out", str(out), "--lambda", str(lam)])
    assert rc == 0
    assert out.read_bytes() == (GOLD / f"{stem}.jhsv").read_bytes()
    assert lam.read_text() == (GOLD / f"{stem}.csv").read_text()


def test_matio_round_trip_and_reference_files(tmp_path):
    g, sig = matio.read_matrix(GOLD / "tg_t3_n64_s5.jhsv")
    assert g.shape == (64, 64) and g.flags.f_contiguous
    assert sig is not None and sig.n == 64
    lam = matio.read_lambda_csv(GOLD / "tg_t3_n64_s5.csv")
    assert sig.n_plus == int((lam > 0).sum())
    p = tmp_path / "x.jhsv"
    matio.write_matrix(p, g, sig)
    assert p.read_bytes() == (GOLD / "tg_t3_n64_s5.jhsv").read_bytes()
    h = np.arange(12.0).reshape(3, 4)
    matio.write_matrix(p, h)
    h2, s2 = matio.read_matrix(p)
    assert s2 is None and np.array_equal(h2, h)
    c = tmp_path / "x.csv"
    matio.write_matrix_csv(c, h)
    assert np.array_equal(matio.read_matrix_csv(c), h)


def test_matio_format_errors(tmp_path):
    p = tmp_path / "bad.jhsv"
    p.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(matio.FormatError):
        matio.read_matrix(p)
    p.write_bytes(struct.pack("<4sIII", b"JHSV", 2, 2, 0) + bytes(8))
    with pytest.raises(matio.FormatError):
        matio.read_matrix(p)
    with pytest.raises(matio.FormatError):
        matio.write_matrix(p, np.zeros((2, 3)), Signature(2, 1))
    assert run(["svd", "run", "--input", str(p)])[0] == 4


def test_host_gen_factor_is_the_reference_construction():
    lam = gen_spectrum(SpectrumSpec(3, 64, 5))
    g, sig = gen_factor(lam, seed=6)
    ref, rsig = matio.read_matrix(GOLD / "tg_t3_n64_s5.jhsv")
    assert np.array_equal(g, ref) and sig == rsig


# ---------------------------------------------------------------------------
# GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name,argv", [
    ("svd_run_t3_n64_w16.json",
     ["svd", "run", "--input", "tg_t3_n64_s5.jhsv", "--lambda", "tg_t3_n64_s5.csv",
      "--width", "16", "--accumulate-v"]),
    ("svd_run_t2_n48_w8_bo_mm.json",
     ["svd", "run", "--input", "tg_t2_n48_s9.jhsv", "--lambda", "tg_t2_n48_s9.csv",
      "--width", "8", "--variant", "bo", "--strategy", "mm"]),
])
def test_svd_run_report_matches_reference(name, argv):
    argv = [str(GOLD / a) if a.endswith((".jhsv", ".csv")) else a for a in argv]
    rc, text = run(argv)
    assert rc == 0
    assert strip_wall(text) == (GOLD / name).read_text()


@pytest.mark.gpu
def test_svd_dist_report_and_trace_match_reference(tmp_path):
    trace = tmp_path / "trace.csv"
    rc, text = run(["svd", "dist", "--input", str(GOLD / "tg_t3_n64_s5.jhsv"), "--lambda",
                    str(GOLD / "tg_t3_n64_s5.csv"), "--width", "8", "--workers", "2",
                    "--accumulate-v", "--trace", str(trace)])
    assert rc == 0
    assert strip_wall(text) == (GOLD / "svd_dist_t3_n64_w8_g2.json").read_text()
    assert trace.read_text() == (GOLD / "svd_dist_trace.csv").read_text()


@pytest.mark.gpu
def test_bench_csv_matches_reference():
    rc, text = run(["bench", "--orders", "32,64", "--types", "1,3", "--variants", "fb,bo",
                    "--width", "16", "--seed", "7"])
    assert rc == 0
    rows = [",".join(line.split(",")[:-1]) for line in text.strip().splitlines()]
    assert "\n".join(rows) + "\n" == (GOLD / "bench_o32-64_t1-3.csv").read_text()


@pytest.mark.gpu
def test_device_file_streaming_round_trip(tmp_path):
    import torch

    G, sig = matio.read_matrix_device(GOLD / "tg_t3_n64_s5.jhsv")
    g, _ = matio.read_matrix(GOLD / "tg_t3_n64_s5.jhsv")
    assert G.is_cuda and torch.equal(G.cpu(), torch.from_numpy(np.ascontiguousarray(g.T)))
    p = tmp_path / "d.jhsv"
    matio.write_matrix_device(p, G, sig)
    assert p.read_bytes() == (GOLD / "tg_t3_n64_s5.jhsv").read_bytes()
    # chunked path: a matrix larger than one staging chunk
    old = matio._CHUNK_BYTES
    try:
        matio._CHUNK_BYTES = 4096
        big = torch.randn(96, 200, dtype=torch.float64, device="cuda")
        matio.write_matrix_device(p, big)
        back, s = matio.read_matrix_device(p)
        assert s is None and torch.equal(back, big)
    finally:
        matio._CHUNK_BYTES = old


@pytest.mark.gpu
@pytest.mark.parametrize("typ,n", [(3, 64), (2, 48)])
def test_device_gen_factor_matches_host_construction(typ, n):
    from paper_1401_2720_b200.testgen import gen_factor_device

    lam = gen_spectrum(SpectrumSpec(typ, n, 11))
    g, sig = gen_factor(lam, seed=12)
    G, dsig = gen_factor_device(lam, seed=12)
    assert dsig == sig
    d = G.cpu().numpy().T
    assert np.max(np.abs(d - g)) <= 1e-13 * np.max(np.abs(g))


@pytest.mark.parametrize("g", [2, 4])
def test_worker_mapping_is_the_references(g):
    from paper_1401_2720_b200 import distsim as D
    from paper_1401_2720_b200.strategy import make_strategy

    ref = json.loads((GOLD / "mappings.json").read_text())[str(g)]
    m = D.default_mapping(make_strategy("rrow", 2 * g))
    assert [[list(pq) for pq in st] for st in m.assignments] == ref["assignments"]
    assert [[list(mv) for mv in st] for st in m.moves] == ref["moves"]
