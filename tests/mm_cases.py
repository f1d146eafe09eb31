"""Seeded Matrix Market texts for the ingest parity tests (test_io.py).

Each case is a byte string. The mix covers what read_matrix_market
(matrix_market.cpp:29-99) accepts and rejects:
  * header variants (case, missing tokens, unsupported object/format/field/symmetry);
  * comment, blank and whitespace-only lines, CRLF endings, tabs, a missing final newline;
  * size-line problems (malformed, missing, negative, too large);
  * entries with values, signs, out-of-range or malformed indices;
  * too few or too many entries, duplicates;
  * symmetric inputs, including non-square ones whose mirror leaves the matrix.
"""
from __future__ import annotations

import random

FIELDS = ["pattern", "real", "integer"]


def _entry(rng: random.Random, rows: int, cols: int, field: str, bad: float) -> str:
    i, j = rng.randint(1, max(rows, 1)), rng.randint(1, max(cols, 1))
    if rng.random() < bad:
        kind = rng.randrange(9)
        if kind == 0:
            i = rng.choice([0, rows + 1, -3])
        elif kind == 1:
            j = rng.choice([0, cols + 1, 10 ** 12])
        elif kind == 2:
            return f"{i}"
        elif kind == 3:
            return "a b"
        elif kind == 4:
            return f"{i}.5 {j}"
        elif kind == 5:
            return f"+{i} {j}"
        elif kind == 6:
            return f"  {i}\t{j}   "
        elif kind == 7:
            return f"{i} {j}x"
        else:
            return f"{i}{'9' * 25} {j}"  # overflows long long
    s = f"{i} {j}"
    if field == "real":
        s += f" {rng.uniform(-10, 10):.3f}"
    elif field == "integer":
        s += f" {rng.randint(-5, 5)}"
    return s


def make_case(seed: int) -> bytes:
    rng = random.Random(seed)
    field = rng.choice(FIELDS)
    sym = rng.random() < 0.3
    rows, cols = rng.randint(0, 12), rng.randint(0, 12)
    if sym and rng.random() < 0.6:
        cols = rows
    banner = "%%MatrixMarket"
    obj, fmt = "matrix", "coordinate"
    symmetry = "symmetric" if sym else "general"
    r = rng.random()
    if r < 0.03:
        banner = "%%matrixmarket"
    elif r < 0.06:
        fmt = "array"
    elif r < 0.08:
        field = "complex"
    elif r < 0.10:
        symmetry = rng.choice(["hermitian", "skew-symmetric"])
    elif r < 0.12:
        obj = "vector"
    elif r < 0.16:
        obj, fmt, field, symmetry = obj.upper(), fmt.title(), field.upper(), symmetry.upper()
    head = f"{banner} {obj} {fmt} {field} {symmetry}"
    if rng.random() < 0.02:
        head = f"{banner} {obj}"  # missing tokens
    lines = [head]
    for _ in range(rng.randint(0, 3)):
        lines.append(rng.choice(["% a comment", "", "   ", "%", "\t"]))
    bad = rng.choice([0.0, 0.0, 0.0, 0.0, 0.05, 0.2])
    n_ent = rng.randint(0, 20) if rows and cols else rng.choice([0, 0, 1])
    ents = []
    for _ in range(n_ent):
        ents.append(_entry(rng, rows, cols, field.lower(), bad))
        if rng.random() < 0.1:
            ents.append(ents[-1])  # duplicate entry
    nnz = declared = len(ents)
    r = rng.random()
    if r < 0.06:
        declared = nnz + rng.randint(1, 3)  # too few entries
    elif r < 0.12:
        declared = max(0, nnz - rng.randint(1, 3))  # data after the declared entries
    size = f"{rows} {cols} {declared}"
    r = rng.random()
    if r < 0.03:
        size = f"{rows} x {declared}"
    elif r < 0.05:
        size = None  # missing size line
    elif r < 0.07:
        size = f"-{rows + 1} {cols} {declared}"
    elif r < 0.09:
        size = f"{2 ** 31} {cols} {declared}"
    elif r < 0.10:
        size = f"{rows} {cols} -2"
    if size is not None:
        lines.append(size)
    for e in ents:
        if rng.random() < 0.1:
            lines.append(rng.choice(["% inner comment", "", "  "]))
        lines.append(e)
    for _ in range(rng.randint(0, 2)):
        lines.append(rng.choice(["% trailing", "", " "]))
    eol = "\r\n" if rng.random() < 0.15 else "\n"
    text = eol.join(lines)
    if rng.random() < 0.85:
        text += eol
    if rng.random() < 0.02:
        text = ""
    return text.encode()


def cases(n: int = 400, seed0: int = 1000) -> list[bytes]:
    out = [make_case(seed0 + k) for k in range(n)]
    # The reference's own test strings (test_csr_graph.cpp:42-112).
    out += [
        b"%%MatrixMarket matrix coordinate pattern general\n2 2 3\n1 1\n2 1\n2 2\n",
        b"%%MatrixMarket matrix coordinate pattern general\n1 1 1\n",
        b"%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 3.5\n2 1 -1.0\n",
        b"%%MatrixMarket matrix array real general\n",
        b"not a header\n",
        b"%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n",
        b"%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n2 2\n",
        b"%%MatrixMarket matrix coordinate pattern symmetric\n2 3 1\n3 1\n",  # mirror leaves a non-square matrix
        b"%%MatrixMarket matrix coordinate pattern symmetric\n3 2 1\n1 3\n",  # row 3 > 2 columns: parse error
    ]
    return out
