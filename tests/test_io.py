"""Dataset ingestion: the native loader
(paper_2204_07485_b200/csrc/io.cpp, bm_parse_file / bm_dataset_load) against
the UNMODIFIED reference loader io::load (io.cpp:82-243, compiled into
oracle/_ref): the same values (bitwise) and the same errors — kind, message,
1-based line and column — on every format, the edge cases the reference
handles (headers, blank lines, CRLF, ragged rows, malformed / missing cells,
non-finite values, column selection, TSPLIB DIMENSION / EOF rules) and a
multi-threaded parse of a large file.  The device half (upload + min-max
normalisation) is in test_gpu_io.py."""
import os

import numpy as np
import pytest

import paper_2204_07485_b200 as bm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D15112 = "/root/reference/proj/data/d15112.tsp"


def _mine(path, **kw):
    try:
        return ("ok", bm.parse_file(path, **kw))
    except bm.ParseError as e:
        return ("parse", str(e), e.line, e.column)
    except bm.ConfigError as e:
        return ("config", str(e), 0, 0)
    except bm.StateError as e:
        return ("state", str(e), 0, 0)


def _same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "ok":
        return a[1].shape == b[1].shape and (a[1].view(np.uint64) == b[1].view(np.uint64)).all()
    return a[1:] == b[1:]


CASES = {
    "plain.csv": ("csv", False, "1,2,3\n4,5,6\n7.25,-8e-3, 9 \n"),
    "header.csv": ("csv", True, "a,b\n1,2\n3,4\n"),
    "blank_lines.csv": ("csv", False, "\n1,2\n\n3,4\n\n"),
    "crlf.csv": ("csv", False, "1,2\r\n3,4\r\n5,6"),
    "no_final_newline.csv": ("csv", False, "1,2\n3,4"),
    "spaces_in_cells.csv": ("csv", False, " 1 ,\t2\n3 , 4\n"),
    "hex_inf_exp.csv": ("csv", False, "0x1p-3,1e300\n-0.0,1.7976931348623157e308\n"),
    "ragged.csv": ("csv", False, "1,2,3\n4,5\n"),
    "ragged_more.csv": ("csv", False, "1,2\n3,4\n5,6,7\n"),
    "malformed.csv": ("csv", False, "1,2\n3,x4\n"),
    "missing.csv": ("csv", False, "1,2\n3,\n"),
    "bad_then_ragged.csv": ("csv", False, "1,2\n3,4,5\n6,zz\n"),
    "cell_before_ragged.csv": ("csv", False, "1,2\nq,4,5\n"),
    "nan.csv": ("csv", False, "1,2\nnan,3\n"),
    "inf.csv": ("csv", False, "1,2\n3,inf\n"),
    "empty.csv": ("csv", False, ""),
    "only_blank.csv": ("csv", False, "\n\n\n"),
    "header_only.csv": ("csv", True, "x,y\n"),
    "blank_header.csv": ("csv", True, "\n1,2\n"),
    "ws.txt": ("whitespace", False, "1 2  3\n\t4\t5 6\n  \n7 8 9   \n"),
    "ws_ragged.txt": ("whitespace", False, "1 2\n3 4 5\n"),
    "ws_header.txt": ("whitespace", True, "x y\n1 2\n"),
    "ws_bad.txt": ("whitespace", False, "1 2\n3 4a\n"),
    "tsp.tsp": ("tsplib", False, "NAME : t\nTYPE : TSP\nDIMENSION : 3\nNODE_COORD_SECTION\n1 1.5 2\n2 3 4\n\n3 5 6\nEOF\n7 8 9\n"),
    "tsp_nodim.tsp": ("tsplib", False, "NODE_COORD_SECTION\n1 1 2\n2 3 4\n"),
    "tsp_dim_mismatch.tsp": ("tsplib", False, "DIMENSION: 5\nNODE_COORD_SECTION\n1 1 2\nEOF\n"),
    "tsp_no_section.tsp": ("tsplib", False, "NAME: x\n1 1 2\n"),
    "tsp_bad_line.tsp": ("tsplib", False, "NODE_COORD_SECTION\n1 1 2 3\n"),
    "tsp_short_line.tsp": ("tsplib", False, "NODE_COORD_SECTION\n1 1\n"),
    "tsp_bad_index.tsp": ("tsplib", False, "NODE_COORD_SECTION\nx 1 2\n"),
    "tsp_empty.tsp": ("tsplib", False, "NODE_COORD_SECTION\nEOF\n"),
    "tsp_bad_dim.tsp": ("tsplib", False, "DIMENSION : abc\nNODE_COORD_SECTION\n1 1 2\n"),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_loader_matches_reference(refo, tmp_path, name):
    fmt, header, text = CASES[name]
    p = tmp_path / name
    p.write_bytes(text.encode())
    assert _same(_mine(p, format=fmt, has_header=header), refo.io_load(p, format=fmt, has_header=header))


@pytest.mark.parametrize("columns", [None, [0], [2, 0], [1, 1, 2], [], [3]])
def test_column_selection_matches_reference(refo, tmp_path, columns):
    p = tmp_path / "cols.csv"
    p.write_text("1,2,3\n4,5,6\n7,8,9\n")
    assert _same(_mine(p, columns=columns), refo.io_load(p, columns=columns))


def test_missing_file_is_state_error(refo, tmp_path):
    p = tmp_path / "nope.csv"
    assert _same(_mine(p), refo.io_load(p))


def test_unknown_format():
    with pytest.raises(bm.ConfigError):
        bm.parse_file("/dev/null", format="xml")


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_large_file_parallel_parse(refo, tmp_path, threads):
    """200k rows: the parallel parse equals the reference bit for bit, and an
    error deep in the file is reported at the same line as the sequential scan."""
    rng = np.random.default_rng(4)
    X = rng.normal(size=(200_000, 7)) * 10 ** rng.uniform(-5, 5, (1, 7))
    p = tmp_path / "big.csv"
    np.savetxt(p, X, delimiter=",", fmt="%.17g")
    got = _mine(p, threads=threads)
    assert _same(got, refo.io_load(p)) and (got[1].view(np.uint64) == X.view(np.uint64)).all()
    lines = p.read_text().splitlines()
    lines[150_001] = lines[150_001].replace(",", ",,", 1)  # a missing value
    lines[170_000] = "1,2"  # a later ragged row
    q = tmp_path / "big_bad.csv"
    q.write_text("\n".join(lines) + "\n")
    assert _same(_mine(q, threads=threads), refo.io_load(q))


@pytest.mark.skipif(not os.path.exists(D15112), reason="reference data absent")
def test_reference_tsplib_instance(refo):
    """The reference's own TSPLIB instance (data/d15112.tsp, registry.json)."""
    got = _mine(D15112, format="tsplib")
    assert got[0] == "ok" and got[1].shape == (15112, 2)
    assert _same(got, refo.io_load(D15112, format="tsplib"))
