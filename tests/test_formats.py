"""File formats and test generation against files the reference itself
wrote (tests/golden/cli/: `jhsvd testgen` outputs of the reference CLI).
CPU tests cover the host paths (testgen files, JHSV / CSV round trips,
format errors); GPU tests the device file streaming and the GPU test
generator."""

import struct
from pathlib import Path

import numpy as np
import pytest

from paper_1401_2720_b200 import matio
from paper_1401_2720_b200.blockkernel import Signature
from paper_1401_2720_b200.testgen import SpectrumSpec, gen_factor, gen_spectrum

GOLD = Path(__file__).resolve().parent / "golden" / "cli"


@pytest.mark.parametrize("typ,n,seed", [(3, 64, 5), (2, 48, 9)])
def test_testgen_files_bitwise(typ, n, seed, tmp_path):
    stem = f"tg_t{typ}_n{n}_s{seed}"
    out, lam = tmp_path / "g.jhsv", tmp_path / "l.csv"
    # the reference `jhsvd testgen` (cli.py:253-262): spectrum seed s, factor seed s + 1
    spec = gen_spectrum(SpectrumSpec(typ, n, seed))
    g, sig = gen_factor(spec, seed=seed + 1)
    matio.write_matrix(out, g, sig)
    matio.write_lambda_csv(lam, spec)
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


def test_host_gen_factor_is_the_reference_construction():
    lam = gen_spectrum(SpectrumSpec(3, 64, 5))
    g, sig = gen_factor(lam, seed=6)
    ref, rsig = matio.read_matrix(GOLD / "tg_t3_n64_s5.jhsv")
    assert np.array_equal(g, ref) and sig == rsig


# ---------------------------------------------------------------------------
# GPU


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
