"""File formats (drop-in for the reference ``jhsvd.matio``, pkg/src/jhsvd/matio.py).

JHSV binary matrix: a 16-byte header (magic "JHSV", u32 rows, u32 cols, u32
flags, little-endian), a u32 n_plus right after it when flags bit 0 is set,
then the entries as little-endian float64 in column-major order
(matio.py:1-7, 28-63).  CSV matrices / eigenvalue vectors use "%.17g", and
strategy tables the reference's text form (matio.py:66-89).

Besides the reference's host functions this module streams JHSV files
straight between disk and HBM: ``read_matrix_device`` maps the file and
uploads it in pinned chunks into the solver's column-major layout (an
(n, m) CUDA tensor), ``write_matrix_device`` the reverse -- the 2-9 GB
inputs of the BASELINE configs never exist as a second host copy.
"""

from __future__ import annotations

import mmap
import struct
from pathlib import Path
from typing import Optional

import numpy as np

from .blockkernel import Signature
from .strategy import PStrategy, dump_strategy, parse_strategy

MAGIC = b"JHSV"
FLAG_SIGNATURE = 1
_CHUNK_BYTES = 64 << 20  # pinned staging chunk for device transfers


class FormatError(ValueError):
    """Malformed or truncated file (matio.py:24-25)."""


def _header(rows: int, cols: int, signature: Optional[Signature]) -> bytes:
    flags = FLAG_SIGNATURE if signature is not None else 0
    h = struct.pack("<4sIII", MAGIC, rows, cols, flags)
    if signature is not None:
        if signature.n != cols:
            raise FormatError("signature order must match the column count")
        h += struct.pack("<I", signature.n_plus)
    return h


def _parse_header(path, data) -> tuple[int, int, int, Optional[Signature]]:
    """(rows, cols, payload offset, signature) from the first bytes."""
    if len(data) < 16 or bytes(data[:4]) != MAGIC:
        raise FormatError(f"{path}: not a JHSV matrix file")
    _, rows, cols, flags = struct.unpack("<4sIII", bytes(data[:16]))
    offset, signature = 16, None
    if flags & FLAG_SIGNATURE:
        if len(data) < 20:
            raise FormatError(f"{path}: truncated signature field")
        (n_plus,) = struct.unpack("<I", bytes(data[16:20]))
        offset = 20
        signature = Signature(cols, n_plus)
    return rows, cols, offset, signature


def write_matrix(path, g, signature: Optional[Signature] = None) -> None:
    """JHSV binary file of g (matio.py:28-41); g may be a numpy array or a
    torch tensor (device tensors are streamed through pinned chunks)."""
    try:
        import torch

        if isinstance(g, torch.Tensor):
            if g.dim() != 2:
                raise FormatError("only 2-d matrices are supported")
            # column-major storage of g (rows, cols) is the (cols, rows) tensor g^T
            write_matrix_device(path, g.t(), signature)
            return
    except ImportError:  # pragma: no cover
        pass
    g = np.asarray(g, dtype=np.float64)
    if g.ndim != 2:
        raise FormatError("only 2-d matrices are supported")
    rows, cols = g.shape
    with open(path, "wb") as fh:
        fh.write(_header(rows, cols, signature))
        fh.write(g.tobytes(order="F"))


def read_matrix(path) -> tuple[np.ndarray, Optional[Signature]]:
    """(g, signature) from a JHSV binary file (matio.py:44-63)."""
    data = Path(path).read_bytes()
    rows, cols, offset, signature = _parse_header(path, data)
    need = rows * cols * 8
    if len(data) - offset != need:
        raise FormatError(f"{path}: expected {need} payload bytes, found {len(data) - offset}")
    flat = np.frombuffer(data, dtype="<f8", offset=offset, count=rows * cols)
    return np.asfortranarray(flat.reshape((rows, cols), order="F")), signature


def read_matrix_device(path, device=None):
    """(G, signature) with G the column-major device storage of the file's
    matrix: an (cols, rows) FP64 CUDA tensor whose row i is column i.  The
    payload is mapped, not read into host memory, and uploaded through
    pinned chunks."""
    import torch

    dev = torch.device("cuda") if device is None else torch.device(device)
    with open(path, "rb") as fh:
        size = Path(path).stat().st_size
        if size < 16:
            raise FormatError(f"{path}: not a JHSV matrix file")
        mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
        try:
            rows, cols, offset, signature = _parse_header(path, mm[:20])
            need = rows * cols * 8
            if size - offset != need:
                raise FormatError(f"{path}: expected {need} payload bytes, "
                                  f"found {size - offset}")
            out = torch.empty((cols, rows), dtype=torch.float64, device=dev)
            flat = out.view(-1)
            src = np.frombuffer(mm, dtype="<f8", count=rows * cols, offset=offset)
            step = max(1, _CHUNK_BYTES // 8)
            pins = [torch.empty(min(step, rows * cols), dtype=torch.float64).pin_memory()
                    for _ in range(2)]
            stream = torch.cuda.current_stream(dev)
            events = [None, None]
            for k, i0 in enumerate(range(0, rows * cols, step)):
                i1 = min(i0 + step, rows * cols)
                buf = pins[k % 2]
                if events[k % 2] is not None:
                    events[k % 2].synchronize()  # the buffer's last copy is done
                buf[: i1 - i0].numpy()[:] = src[i0:i1]
                flat[i0:i1].copy_(buf[: i1 - i0], non_blocking=True)
                events[k % 2] = torch.cuda.Event()
                events[k % 2].record(stream)
            torch.cuda.current_stream(dev).synchronize()
            del src
        finally:
            mm.close()
    return out, signature


def write_matrix_device(path, G, signature: Optional[Signature] = None) -> None:
    """JHSV file of the matrix whose column-major storage is the (cols, rows)
    tensor G (the solver's layout), streamed through pinned chunks."""
    import torch

    if G.dim() != 2:
        raise FormatError("only 2-d matrices are supported")
    cols, rows = (int(s) for s in G.shape)
    Gc = G.contiguous()
    flat = Gc.reshape(-1)
    step = max(1, _CHUNK_BYTES // 8)
    with open(path, "wb") as fh:
        fh.write(_header(rows, cols, signature))
        if Gc.device.type != "cuda":
            fh.write(flat.to(torch.float64).numpy().astype("<f8", copy=False).tobytes())
            return
        pin = torch.empty(min(step, rows * cols), dtype=torch.float64).pin_memory()
        for i0 in range(0, rows * cols, step):
            i1 = min(i0 + step, rows * cols)
            pin[: i1 - i0].copy_(flat[i0:i1])
            fh.write(pin[: i1 - i0].numpy().tobytes())


def write_matrix_csv(path, g) -> None:
    np.savetxt(path, np.asarray(g, dtype=np.float64), delimiter=",", fmt="%.17g")


def read_matrix_csv(path) -> np.ndarray:
    g = np.loadtxt(path, delimiter=",", ndmin=2)
    return np.asfortranarray(g.astype(np.float64))


def write_lambda_csv(path, lam) -> None:
    np.savetxt(path, np.asarray(lam, dtype=np.float64), delimiter=",", fmt="%.17g")


def read_lambda_csv(path) -> np.ndarray:
    lam = np.loadtxt(path, delimiter=",")
    return np.atleast_1d(lam.astype(np.float64))


def save_strategy(path, strat: PStrategy) -> None:
    Path(path).write_text(dump_strategy(strat))


def load_strategy(path, kind: str = "custom") -> PStrategy:
    return parse_strategy(Path(path).read_text(), kind=kind)
