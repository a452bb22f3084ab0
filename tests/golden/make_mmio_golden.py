"""Freeze the REFERENCE's Matrix Market reader outputs (tests/golden/mmio_cases.json).

Test infrastructure: imports ``maskmul.mmio.read_matrix_market``
(pkg/src/maskmul/mmio.py:27-101) from /root/reference (build container only)
and records, for each text below, either the canonical CSR digest (the
convention of make_golden.py) or the exception class and line number.  The
texts are the reference's own test_mmio.py cases plus seeded variations of
formatting (comments, blank lines, CRLF, tabs, signs, underscores, exponent
forms, 17-digit reprs, inf/nan, duplicates, symmetric) and one error of each
kind at a known line.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mmio_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from maskmul.mmio import read_matrix_market  # noqa: E402

from golden_util import GOLDEN, digest_csr  # noqa: E402

H = "%%MatrixMarket matrix coordinate"

HAND = {
    # pkg/tests/test_mmio.py cases
    "pattern_symmetric": f"{H} pattern symmetric\n2 2 1\n2 1\n",
    "real_general": f"{H} real general\n3 3 3\n1 1 1.5\n2 3 -2.0\n3 1 4\n",
    "integer_field": f"{H} integer general\n2 2 1\n1 2 7\n",
    "zero_index": f"{H} pattern general\n2 2 1\n0 1\n",
    "bad_banner": "%%NotMatrixMarket blah\n1 1 0\n",
    "complex_field": f"{H} complex general\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n1 1\n1.0\n",
    "too_few": f"{H} real general\n2 2 2\n1 1 1\n",
    "too_many": f"{H} real general\n2 2 1\n1 1 1\n2 2 1\n",
    "comments_blank": f"{H} real general\n% a comment\n\n2 2 2\n% another\n1 1 3\n\n2 2 4\n",
    "sym_diag_once": f"{H} real symmetric\n2 2 2\n1 1 5\n2 1 3\n",
    "duplicates": f"{H} integer general\n2 2 2\n1 1 2\n1 1 3\n",
    # further edge cases of the same code path
    "empty_file": "",
    "no_size_line": f"{H} real general\n% only a comment\n\n",
    "size_two_fields": f"{H} real general\n2 2\n",
    "size_non_int": f"{H} real general\n2 x 1\n1 1 1\n",
    "size_negative": f"{H} real general\n-2 2 0\n",
    "bad_symmetry": f"{H} real hermitian\n1 1 0\n",
    "short_header": f"{H} real\n1 1 0\n",
    "zero_entries": f"{H} real general\n3 4 0\n",
    "zero_dims": f"{H} pattern general\n0 0 0\n",
    "entry_too_few_fields": f"{H} real general\n2 2 1\n1 1\n",
    "pattern_extra_tokens": f"{H} pattern general\n2 2 1\n1 2 99 junk\n",
    "index_float": f"{H} integer general\n2 2 1\n1.0 1 3\n",
    "index_out_of_range": f"{H} integer general\n2 3 2\n1 1 1\n2 4 1\n",
    "row_out_of_range": f"{H} integer general\n2 3 1\n3 1 1\n",
    "bad_real": f"{H} real general\n2 2 1\n1 1 abc\n",
    "bad_integer": f"{H} integer general\n2 2 1\n1 1 2.5\n",
    "hex_real_rejected": f"{H} real general\n1 1 1\n1 1 0x1p3\n",
    "crlf": f"{H} real general\r\n2 2 2\r\n1 1 0.5\r\n2 2 -1e-3\r\n",
    "tabs_spaces": f"  {H} integer general  \n\t2\t2\t2\n  1\t 2   -3  \n2 1 +4\n",
    "tabs_spaces_ok": f"{H}   integer\tgeneral  \n\t2\t2\t2\n  1\t 2   -3  \n2 1 +4\n",
    "signs_underscores": f"{H} integer general\n1_0 1_0 2\n+1 +1_0 1_000\n0_10 1 -7\n",
    "bad_underscore": f"{H} integer general\n2 2 1\n1 1 1__0\n",
    "real_forms": (f"{H} real general\n1 8 8\n1 1 1.\n1 2 .5\n1 3 -0.0\n1 4 1E+2\n1 5 2e-320\n"
                   f"1 6 inf\n1 7 -Infinity\n1 8 1_0.2_5e0_1\n"),
    "real_overflow_to_inf": f"{H} real general\n1 1 1\n1 1 1e400\n",
    "no_trailing_newline": f"{H} real general\n2 2 1\n2 2 7.25",
    "count_short_no_newline": f"{H} real general\n2 2 3\n2 2 7.25\n1 1 1",
    "comment_after_entries": f"{H} real general\n2 2 1\n2 2 7.25\n% trailing\n\n",
    "error_beats_count": f"{H} real general\n2 2 3\n1 1 1\n1 3 1\n",
    "more_than_then_bad": f"{H} real general\n2 2 1\n1 1 1\nfoo bar baz\n",
    "symmetric_integer_dups": f"{H} integer symmetric\n3 3 4\n2 1 1\n1 2 10\n3 3 2\n3 3 5\n",
}


def random_text(rng, field: str, symmetric: bool, n: int, nnz: int, style: int) -> str:
    rows = rng.integers(1, n + 1, nnz)
    cols = rng.integers(1, n + 1, nnz)
    if symmetric:
        lo = np.minimum(rows, cols)
        hi = np.maximum(rows, cols)
        rows, cols = hi, lo
    out = [f"{H} {field} {'symmetric' if symmetric else 'general'}\n", "% generated\n", f"{n} {n} {nnz}\n"]
    for t in range(nnz):
        line = f"{rows[t]} {cols[t]}"
        if field == "real":
            x = float(rng.standard_normal() * 10.0 ** rng.integers(-30, 30))
            forms = [repr(x), f"{x:.17g}", f"{x:.3e}", f"{x:g}", f"{x:.17E}"]
            line += " " + forms[(style + t) % len(forms)]
        elif field == "integer":
            line += f" {int(rng.integers(-10**12, 10**12))}"
        if style == 1 and t % 7 == 0:
            out.append("% interleaved comment\n\n")
        if style == 2:
            line = "  " + line.replace(" ", "\t") + " \r"
        out.append(line + "\n")
    return "".join(out)


def expected(text: str):
    with tempfile.NamedTemporaryFile("wb", suffix=".mtx", delete=False) as fh:
        fh.write(text.encode("ascii"))
        path = fh.name
    try:
        m = read_matrix_market(path)
    except Exception as e:  # noqa: BLE001 - recorded as the expected outcome
        return {"error": type(e).__name__, "lineno": getattr(e, "lineno", None)}
    finally:
        os.unlink(path)
    return {"shape": [m.nrows, m.ncols], "nnz": int(m.nnz), "dtype": str(m.values.dtype),
            "digest": digest_csr(m.row_ptr, m.col_idx, m.values)}


def main() -> None:
    cases = []
    for name, text in HAND.items():
        cases.append({"name": name, "text": text, "expect": expected(text)})
    rng = np.random.default_rng(777)
    for field in ("real", "integer", "pattern"):
        for symmetric in (False, True):
            for style in range(3):
                n = int(rng.integers(1, 40))
                text = random_text(rng, field, symmetric, n, int(rng.integers(0, 120)), style)
                cases.append({"name": f"random_{field}_{'sym' if symmetric else 'gen'}_{style}",
                              "text": text, "expect": expected(text)})
    path = os.path.join(GOLDEN, "mmio_cases.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_mmio_golden.py (reference maskmul.mmio)",
                   "cases": cases}, fh, indent=0)
    print(f"wrote {len(cases)} cases to {path}")


if __name__ == "__main__":
    main()
