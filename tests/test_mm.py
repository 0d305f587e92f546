"""Matrix Market ingest (io.hpp:17-123) -- host parser in libgfb (mm.cu),
checked on CPU against the reference's own test_io.cpp cases and against the
unmodified reference parser (oracle/_ref ref_mm_parse) on generated files,
valid and malformed: same edges in the same order, same error line and
message."""
import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

HDR = "%%MatrixMarket matrix coordinate real general\n"


def edges_equal(el, want):
    return el.edges == [(s, d, float(w)) for s, d, w in want]


# ---- test_io.cpp:24-117, restated -----------------------------------------
def test_general_real():  # :24-29
    el = gb.parse_matrix_market(HDR + "3 3 2\n1 2 1.0\n2 3 2.0\n")
    assert el.num_vertices == 3 and edges_equal(el, [(0, 1, 1.0), (1, 2, 2.0)])


def test_pattern_symmetric_expand():  # :31-41
    text = "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 1\n1 2\n"
    assert edges_equal(gb.parse_matrix_market(text, expand_symmetric=True),
                       [(0, 1, 1.0), (1, 0, 1.0)])
    assert edges_equal(gb.parse_matrix_market(text), [(0, 1, 1.0)])


def test_symmetric_diagonal_once():  # :43-51
    el = gb.parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n"
                                "1 1 3.0\n2 1 1.0\n", expand_symmetric=True)
    assert edges_equal(el, [(0, 0, 3.0), (1, 0, 1.0), (0, 1, 1.0)])


def test_integer_and_zero_weights():  # :53-58
    el = gb.parse_matrix_market("%%MatrixMarket matrix coordinate integer general\n2 2 2\n"
                                "1 2 0\n2 1 7\n")
    assert el.w.tolist() == [0.0, 7.0]


def test_force_unit_weights():  # :60-66
    el = gb.parse_matrix_market(HDR + "2 2 1\n1 2 5.5\n", force_unit_weights=True)
    assert el.w.tolist() == [1.0]


def test_comments_skipped():  # :68-72
    el = gb.parse_matrix_market(HDR + "% a comment\n2 2 1\n% another\n1 2 1.5\n")
    assert len(el.edges) == 1


@pytest.mark.parametrize("text,line,frag", [
    ("%%NotMatrixMarket whatever\n", 1, "malformed header"),                          # :75-82
    (HDR + "5 5 5\n1 2 1\n2 3 1\n3 4 1\n4 5 1\n", 6, "declares 5"),               # :83-93
    (HDR + "2 2 1\n1 2 1\n2 1 1\n", 4, "found more"),                             # :94-98
    (HDR + "2 2 1\n1 3 1.0\n", 3, "index out of declared bounds"),                # :99-107
    (HDR + "2 2 1\n1 2 -1.0\n", 3, "negative weight"),                            # :108-111
    (HDR + "2 3 1\n1 2 1.0\n", 2, "rectangular"),                                 # :112-116
])
def test_rejections_carry_line_numbers(text, line, frag):
    with pytest.raises(gb.ParseError) as e:
        gb.parse_matrix_market(text)
    assert e.value.line == line and frag in str(e.value)
    assert str(e.value).startswith(f"line {line}: ")


def test_declared_five_found_four_message():  # :88-91
    with pytest.raises(gb.ParseError) as e:
        gb.parse_matrix_market(HDR + "5 5 5\n1 2 1\n2 3 1\n3 4 1\n4 5 1\n")
    assert "declares 5" in str(e.value) and "found 4" in str(e.value)


def test_write_distances():  # :119-130
    assert gb.write_distances([0.0, 1.0, 3.0], [gb.NIL, 0, 1]) == "0 0 -\n1 1 0\n2 3 1\n"
    assert gb.write_distances([0.0, float("inf")], [gb.NIL, gb.NIL]) == "0 0 -\n1 inf -\n"


# ---- against the unmodified reference parser --------------------------------
def _ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")


def _same(text, **kw):
    want = O.ref_mm_parse(text, **kw)
    try:
        el = gb.parse_matrix_market(text, **kw)
    except gb.ParseError as e:
        assert want[0] == "error", (str(e), want)
        assert (e.line, str(e)) == (want[1], want[2])
        return
    assert want[0] != "error", want
    n, s, d, w = want
    assert el.num_vertices == n
    assert np.array_equal(el.src, s) and np.array_equal(el.dst, d)
    assert np.array_equal(el.w.view(np.uint64), w.view(np.uint64))


def _gen_file(rng, n, k, field, sym, comments, crlf):
    lines = [f"%%MatrixMarket matrix coordinate {field} {sym}"]
    if comments:
        lines.append("% generated")
    lines.append(f"{n} {n} {k}")
    for _ in range(k):
        i, j = rng.integers(1, n + 1, 2)
        if field == "pattern":
            lines.append(f"{i} {j}")
        elif field == "integer":
            lines.append(f"{i} {j} {rng.integers(0, 1000)}")
        else:
            lines.append(f"{i}\t{j}  {rng.random() * 10.0 ** int(rng.integers(-5, 5)):.17g}")
        if comments and rng.random() < 0.1:
            lines.append("% c")
        if rng.random() < 0.05:
            lines.append("")
    sep = "\r\n" if crlf else "\n"
    return sep.join(lines) + sep


def test_generated_files_match_reference():
    _ref()
    rng = np.random.default_rng(11)
    for t in range(60):
        text = _gen_file(rng, int(rng.integers(1, 300)), int(rng.integers(0, 400)),
                         ["real", "integer", "pattern"][t % 3], ["general", "symmetric"][t % 2],
                         t % 4 == 0, t % 5 == 0)
        for kw in (dict(), dict(expand_symmetric=True), dict(force_unit_weights=True)):
            _same(text, **kw)


def test_malformed_files_match_reference():
    _ref()
    rng = np.random.default_rng(12)
    base = _gen_file(rng, 50, 40, "real", "general", True, False).split("\n")
    mutations = ["1 2", "x 2 3", "1 y 3", "0 1 1.0", "51 1 1.0", "1 2 -0.5", "1 2 nan",
                 "1 2 inf", "1 2 1e400", "1 2 +3.5", "1.5 2 3", " 3 4 5 6", "%%", "", "\t",
                 "1 2 .5", "1 2 5.", "1 2 -0", "7 7 1e-320"]
    for t in range(120):
        lines = list(base)
        pos = int(rng.integers(1, len(lines)))
        lines.insert(pos, mutations[t % len(mutations)])
        if t % 7 == 0:
            lines[0] = lines[0].replace("general", ["hermitian", "skew", "General"][t % 3])
        if t % 11 == 0:
            lines[0] = lines[0].replace("real", "complex")
        _same("\n".join(lines))
    for text in ("", "\n", "%%MatrixMarket matrix coordinate real general\n",
                 "%%MatrixMarket matrix coordinate real general\n% only comments\n",
                 "%%MatrixMarket matrix coordinate real general\n2 2\n",
                 "%%MatrixMarket matrix array real general\n2 2 0\n",
                 "%%MatrixMarket matrix coordinate real general\n0 0 0\n"):
        _same(text)
