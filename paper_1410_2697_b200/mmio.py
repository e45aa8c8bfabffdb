"""Matrix Market interchange and row scaling (host I/O around the hot path).

Same file format, validation rules and error texts as the reference's
``load_matrix_market`` / ``write_matrix_market`` / ``row_scale``
(sparse.py:142-274), so the identical matrix reaches both implementations
(SURVEY 8(f)-2). Parsing is vectorised: the reference checks entries one line
at a time; here the checks run on whole arrays and the FIRST offending line is
reported, with the reference's precedence inside one line (malformed, out of
range, duplicate, too many entries, symmetric upper-triangle entry).
"""
from __future__ import annotations

import numpy as np

from .sparse import SparseMatrix


class _Fail(ValueError):
    pass


def load_matrix_market(path):
    """Read a coordinate real (general or symmetric) Matrix Market file.

    Symmetric files must store the lower triangle; the pattern is expanded to
    full storage and the symmetric flag set. Indices become 0-based.
    """
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.read().splitlines()

    def fail(lineno, msg):
        raise ValueError(f"{path}:{lineno}: {msg}")

    if not lines:
        fail(1, "empty file")
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket":
        fail(1, "missing '%%MatrixMarket' header")
    obj, fmt, field, symmetry = (t.lower() for t in head[1:])
    if obj != "matrix" or fmt != "coordinate":
        fail(1, f"unsupported header '{lines[0]}' (need coordinate matrix)")
    if field != "real":
        fail(1, f"unsupported field '{field}' (only real is accepted)")
    if symmetry not in ("general", "symmetric"):
        fail(1, f"unsupported symmetry '{symmetry}'")
    sym = symmetry == "symmetric"

    # size line: the first line after the header that is neither blank nor a comment
    k = 1
    while k < len(lines) and (not lines[k].strip() or lines[k].strip().startswith("%")):
        k += 1
    if k >= len(lines):
        fail(max(k, 2) if len(lines) > 1 else 1, "missing size line")
    size_line = lines[k].strip()
    size = size_line.split()
    try:
        if len(size) != 3:
            raise _Fail
        n_rows, n_cols, n_entries = (int(t) for t in size)
    except (_Fail, ValueError):
        fail(k + 1, f"malformed size line '{size_line}'")
    if sym and n_rows != n_cols:
        fail(k + 1, "symmetric matrix must be square")

    # entry lines (blank lines skipped; a comment here is a malformed entry, as in the reference)
    body = [(ln, t) for ln, t in ((j + 1, lines[j].strip()) for j in range(k + 1, len(lines))) if t]
    m = len(body)
    rows = np.empty(m, dtype=np.int64)
    cols = np.empty(m, dtype=np.int64)
    vals = np.empty(m, dtype=np.float64)
    bad_parse = m  # first entry that does not parse
    for q, (ln, t) in enumerate(body):
        parts = t.split()
        try:
            if len(parts) != 3:
                raise _Fail
            rows[q] = int(parts[0])
            cols[q] = int(parts[1])
            vals[q] = float(parts[2])
        except (_Fail, ValueError):
            bad_parse = q
            break
    ok = slice(0, bad_parse)
    r, c = rows[ok], cols[ok]
    out_range = np.flatnonzero((r < 1) | (r > n_rows) | (c < 1) | (c > n_cols))
    first_range = int(out_range[0]) if out_range.size else m
    # duplicates: the second occurrence of a (row, col) key is the offending line
    lim = min(bad_parse, first_range)
    key = (r[:lim] - 1) * max(n_cols, 1) + (c[:lim] - 1)
    order = np.argsort(key, kind="stable")
    sk = key[order]
    dup_pos = order[1:][sk[1:] == sk[:-1]]
    first_dup = int(dup_pos.min()) if dup_pos.size else m
    first_upper = m
    if sym:
        up = np.flatnonzero(c[:lim] > r[:lim])
        first_upper = int(up[0]) if up.size else m
    over = n_entries if m > n_entries else m  # the entry that exceeds the declared count
    # per line the reference checks: parse, range, duplicate, count, upper triangle
    cands = [(bad_parse, 0), (first_range, 1), (first_dup, 2), (over, 3), (first_upper, 4)]
    q, kind = min(cands)
    if q < m:
        ln, t = body[q]
        if kind == 0:
            fail(ln, f"malformed entry line '{t}'")
        if kind == 1:
            fail(ln, f"entry ({rows[q]}, {cols[q]}) out of range for {n_rows}x{n_cols}")
        if kind == 2:
            fail(ln, f"duplicate entry ({rows[q]}, {cols[q]})")
        if kind == 3:
            raise ValueError(f"{path}: entry count mismatch: header declares {n_entries}, file has more")
        fail(ln, "symmetric file stores an entry above the diagonal")
    if m != n_entries:
        raise ValueError(f"{path}: entry count mismatch: header declares {n_entries}, file has {m}")
    i0, j0 = rows - 1, cols - 1
    if sym:
        off = i0 != j0
        i0, j0, vals = (np.concatenate([i0, j0[off]]), np.concatenate([j0, i0[off]]),
                        np.concatenate([vals, vals[off]]))
    return SparseMatrix.from_triplets(n_rows, n_cols, i0, j0, vals, symmetric=sym)


def write_matrix_market(A, path):
    """Coordinate format, 1-based ASCII; a symmetric matrix is written with a
    symmetric header and its lower triangle only (round trips reproduce the
    entry multiset). Values in Python's shortest round-trip repr."""
    coo = A._csc.tocoo()
    rows, cols, vals = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
    if A.symmetric:
        keep = rows >= cols
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate real {'symmetric' if A.symmetric else 'general'}\n")
        fh.write(f"{A.n_rows} {A.n_cols} {len(vals)}\n")
        fh.write("".join(f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(rows.tolist(), cols.tolist(),
                                                                                 vals.tolist())))


class ScalingRecord:
    """Per-row divisors applied by :func:`row_scale` (sparse.py:135-139)."""

    def __init__(self, row_scales):
        self.row_scales = row_scales


def row_scale(A, b):
    """Divide each row of ``A`` (and ``b``) by its largest absolute entry; the
    result never carries the symmetric flag (sparse.py:252-274)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != A.n_rows:
        raise ValueError("right-hand side length does not match matrix rows")
    csr = A.to_csr()
    csr.sort_indices()
    counts = np.diff(csr.indptr)
    empty = np.flatnonzero(counts == 0)
    mx = np.zeros(A.n_rows)
    nz = counts > 0
    if nz.any():
        mx[nz] = np.maximum.reduceat(np.abs(csr.data), csr.indptr[:-1][nz])
    bad = np.flatnonzero(mx == 0.0)
    if empty.size or bad.size:
        i = int(min(empty.min() if empty.size else A.n_rows, bad.min() if bad.size else A.n_rows))
        raise ValueError(f"row {i} has no nonzero entries")
    csr.data /= np.repeat(mx, counts)
    return SparseMatrix(csr.tocsc()), b / mx, ScalingRecord(mx)
