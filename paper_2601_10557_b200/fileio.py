"""On-disk formats of the reference (docs/FORMATS.md), so both solvers read the
same input bytes and emit byte-compatible outputs.

* PCHB (Hamiltonian blocks), PCHV (eigenvectors): little endian, column major;
  ``read_pchb(..., device=...)`` streams the blocks straight into the device
  ``[A | B]`` buffer without building host complex128 copies.
* Matrix Market array (complex general), eigenvalues / trace CSV, manifest —
  17 significant digits so write -> read -> write is byte identical.
Host-side I/O only; nothing here is on the GPU hot path.
"""

from __future__ import annotations

import hashlib
import json
import struct
from datetime import datetime, timezone
from pathlib import Path

import numpy as np

from . import __version__
from .errors import ValidationError
from .hamiltonian import BseHamiltonian, Definiteness, as_complex_matrix, colmajor_empty

PCHB_HEADER = struct.Struct("<4sIQ")     # magic, version, m
PCHV_HEADER = struct.Struct("<4sIQQ")    # magic, version, n, k
FORMAT_VERSION = 1
MM_BANNER = "%%MatrixMarket matrix array complex general"


def digest64(path) -> str:
    """blake2b with an 8-byte digest over the raw file bytes (FORMATS.md)."""
    h = hashlib.blake2b(digest_size=8)
    with open(path, "rb") as fh:
        while chunk := fh.read(1 << 22):
            h.update(chunk)
    return h.hexdigest()


# ------------------------------------------------------------------------------------------- PCHB
def write_pchb(path, ham: BseHamiltonian) -> None:
    a, b = ham.host_blocks()
    with open(path, "wb") as fh:
        fh.write(PCHB_HEADER.pack(b"PCHB", FORMAT_VERSION, ham.m))
        for blk in (a, b):
            np.asfortranarray(blk, dtype="<c16").T.tofile(fh)  # column-major bytes


def _pchb_header(fh) -> int:
    raw = fh.read(PCHB_HEADER.size)
    if len(raw) != PCHB_HEADER.size:
        raise ValidationError("truncated PCHB header")
    magic, version, m = PCHB_HEADER.unpack(raw)
    if magic != b"PCHB":
        raise ValidationError(f"not a PCHB file (magic {magic!r})")
    if version != FORMAT_VERSION:
        raise ValidationError(f"unsupported PCHB version {version}")
    return int(m)


def read_pchb(path, device=None, definiteness: Definiteness = Definiteness.UNKNOWN) -> BseHamiltonian:
    """Host BseHamiltonian (reference semantics: validated / symmetrised), or with ``device``
    a device-born one filled column block by column block (no host complex copy of A|B)."""
    with open(path, "rb") as fh:
        m = _pchb_header(fh)
        count = m * m
        if device is None:
            a = np.fromfile(fh, dtype="<c16", count=count)
            b = np.fromfile(fh, dtype="<c16", count=count)
            if a.size != count or b.size != count:
                raise ValidationError("truncated PCHB payload")
            return BseHamiltonian(a.reshape((m, m), order="F"), b.reshape((m, m), order="F"), definiteness)
        import torch

        ab = colmajor_empty(m, 2 * m, device)
        cols = max(1, (1 << 27) // max(16 * m, 1))  # ~128 MB slabs
        staging = torch.empty((cols, m), dtype=torch.complex128, pin_memory=True)
        for c0 in range(0, 2 * m, cols):
            c1 = min(2 * m, c0 + cols)
            got = fh.readinto(memoryview(staging.numpy()[: c1 - c0]).cast("B"))
            if got != 16 * m * (c1 - c0):
                raise ValidationError("truncated PCHB payload")
            ab[:, c0:c1].copy_(staging[: c1 - c0].T, non_blocking=False)
        ham = BseHamiltonian.from_device(ab, definiteness)
        # device-born input: the reference's symmetry repair (hamiltonian.py:45-60) is checked on
        # the device; reject beyond 1e-12 x scale like the host constructor
        a_d, b_d = ab[:, :m], ab[:, m:]
        scale = float(torch.max(torch.abs(ab)).item()) if m else 0.0
        da = float(torch.max(torch.abs(a_d - a_d.conj().T)).item()) if m else 0.0
        db = float(torch.max(torch.abs(b_d - b_d.T)).item()) if m else 0.0
        if max(da, db) > 1e-12 * scale:
            raise ValidationError(f"blocks violate hermiticity/symmetry beyond tolerance ({max(da, db):.3e})")
        if da:
            a_d.copy_((a_d + a_d.conj().T) / 2)
        if db:
            b_d.copy_((b_d + b_d.T) / 2)
        return ham


# ------------------------------------------------------------------------------------------- PCHV
def write_pchv(path, vectors) -> None:
    v = vectors.T.contiguous().cpu().numpy().T if hasattr(vectors, "cpu") else as_complex_matrix(vectors, "vectors")
    with open(path, "wb") as fh:
        fh.write(PCHV_HEADER.pack(b"PCHV", FORMAT_VERSION, v.shape[0], v.shape[1]))
        np.asfortranarray(v, dtype="<c16").T.tofile(fh)


def read_pchv(path) -> np.ndarray:
    with open(path, "rb") as fh:
        raw = fh.read(PCHV_HEADER.size)
        magic, version, n, k = PCHV_HEADER.unpack(raw)
        if magic != b"PCHV":
            raise ValidationError(f"not a PCHV file (magic {magic!r})")
        if version != FORMAT_VERSION:
            raise ValidationError(f"unsupported PCHV version {version}")
        data = np.fromfile(fh, dtype="<c16", count=n * k)
    return np.asfortranarray(data.reshape((n, k), order="F"))


# ---------------------------------------------------------------------------------- Matrix Market
def write_matrix_market(path, matrix, comment: str | None = None) -> None:
    a = as_complex_matrix(matrix, "matrix")
    lines = [MM_BANNER]
    if comment:
        lines += [f"%{c}" for c in comment.splitlines()]
    lines.append(f"{a.shape[0]} {a.shape[1]}")
    flat = a.reshape(-1, order="F")
    lines += [f"{z.real:.17e} {z.imag:.17e}" for z in flat]
    Path(path).write_text("\n".join(lines) + "\n")


def read_matrix_market(path) -> np.ndarray:
    with open(path) as fh:
        banner = fh.readline().strip()
        if banner.lower().split() != MM_BANNER.lower().split():
            raise ValidationError(f"unsupported Matrix Market header: {banner!r}")
        line = fh.readline()
        while line.startswith("%"):
            line = fh.readline()
        try:
            rows, cols = map(int, line.split())
        except ValueError as exc:
            raise ValidationError(f"malformed size line: {line!r}") from exc
        vals = np.loadtxt(fh, dtype=np.float64, ndmin=2)
    if vals.shape != (rows * cols, 2):
        raise ValidationError(f"expected {rows * cols} complex entries, got {vals.shape[0]}")
    return np.asfortranarray((vals[:, 0] + 1j * vals[:, 1]).reshape((rows, cols), order="F"))


# ------------------------------------------------------------------------------------------- CSVs
def write_eigenvalues_csv(path, lambdas, residual_norms, input_digest: str, converged: bool = True) -> None:
    rows = [
        "# bsesolve eigenvalues v1", "# manifest: manifest.json", f"# input_digest: {input_digest}",
        f"# converged: {'true' if converged else 'false'}", "index,eigenvalue,residual",
    ]
    rows += [f"{i},{lam:.17g},{res:.17g}" for i, (lam, res) in enumerate(zip(np.asarray(lambdas),
                                                                          np.asarray(residual_norms)))]
    Path(path).write_text("\n".join(rows) + "\n")


def write_trace_csv(path, result, input_digest: str) -> None:
    rows = [
        "# bsesolve trace v1", "# manifest: manifest.json", f"# input_digest: {input_digest}",
        f"# mu_1: {result.bounds.mu_1:.17g}", f"# mu_n: {result.bounds.mu_n:.17g}",
        f"# converged: {'true' if result.converged else 'false'}",
        "iter,locked,k,max_res,min_res_unlocked,mu_nevex,variant,lambda_min_M,flops",
    ]
    rows += [f"{t.it},{t.locked},{t.k},{t.max_res:.17g},{t.min_res_unlocked:.17g},{t.mu_nevex:.17g},"
             f"{t.variant},{t.lambda_min_m:.17g},{t.flops:.0f}" for t in result.trace]
    Path(path).write_text("\n".join(rows) + "\n")


def write_manifest(path, command: str, config: dict, inputs: dict, outputs: list, seed) -> None:
    doc = {"tool": "bsesolve", "version": __version__, "implementation": "paper_2601_10557_b200 (B200)",
           "command": command, "config": config, "inputs": inputs, "outputs": outputs, "seed": seed,
           "written_utc": datetime.now(timezone.utc).isoformat()}
    Path(path).write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")
