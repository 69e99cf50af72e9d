"""Ingest: the loaders of csrc/io.cpp against the
reference's own load_points / load_obj_projected (datagen.hpp:111-168, run
from oracle/_ref) on the same files: identical coordinates bit for bit,
identical error kinds and messages; and the GSCANSOA binary round trip."""
import numpy as np
import pytest

import oracle

CASES_XY = {
    "plain": "1 2\n3 4\n",
    "comments_blank_ws": "# header\n\n  1.5\t-2.25  \r\n\t# indented comment\n7e-300 1e300\n",
    "crlf": "1 2\r\n3 4\r\n",
    "exp_forms": "1E5 -0.0\n.5 5.\n-1e-5 2.5e+3\n",
    "no_newline": "8 9",
    "trailing": "1 2 3\n",
    "bad_x": "x 2\n",
    "missing_y": "1\n",
    "plus_sign": "+1 2\n",
    "nonfinite": "1 inf\n",
    "nan": "nan 1\n",
    "empty": "",
    "only_comments": "# a\n\n# b\n",
    "late_error": "1 2\n3 4\n5 6 junk\n",
}
CASES_OBJ = {
    "vertices": "v 1 2 3\nv 4 5 6\n",
    "mixed": "# obj\nvt 0.5 0.5\nvn 0 0 1\nv 1 2 3\nf 1 2 3\nv\t-1\t-2\n",
    "no_z_and_junk": "v 1 2\nv 3 4 5 6 extra\n",
    "v_prefix_token": "vx 1 2\nv 7 8\n",
    "bad_vertex": "v 1 y\n",
    "no_vertices": "vt 1 2\nf 1 2 3\n",
    "nonfinite": "v nan 1 2\n",
}


def _ours(path, fmt):
    from paper_1508_05931_b200 import EmptyInput, IoError, ParseError, load_points
    try:
        xs, ys = load_points(path, fmt)
        return 0, xs, ys, ""
    except ParseError as e:
        return 1, None, None, str(e)
    except IoError as e:
        return 2, None, None, str(e)
    except EmptyInput as e:
        return 3, None, None, str(e)


def _check(tmp_path, name, text, obj):
    p = tmp_path / f"{name}.{'obj' if obj else 'txt'}"
    p.write_bytes(text.encode())
    rc_r, xr, yr, mr = oracle.ref_load(p, obj)
    rc_o, xo, yo, mo = _ours(p, "obj" if obj else "xy")
    assert rc_o == rc_r, (name, rc_o, rc_r, mo, mr)
    assert mo == mr, (name, mo, mr)
    if rc_r == 0:
        assert np.array_equal(xo.view(np.uint64), xr.view(np.uint64)), name
        assert np.array_equal(yo.view(np.uint64), yr.view(np.uint64)), name


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", sorted(CASES_XY))
def test_xy_loader_matches_reference(tmp_path, name):
    _check(tmp_path, name, CASES_XY[name], False)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", sorted(CASES_OBJ))
def test_obj_loader_matches_reference(tmp_path, name):
    _check(tmp_path, name, CASES_OBJ[name], True)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_random_text_round_trip_matches_reference(tmp_path):
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.standard_normal(3000) * 10.0 ** rng.integers(-300, 290, 3000),
                         [0.0, -0.0, 5e-324, 1.7976931348623157e308]])
    ys = rng.uniform(-1, 1, xs.size)
    text = "".join(f"{float(x)!r} {float(y)!r}\n" for x, y in zip(xs, ys))
    _check(tmp_path, "random", text, False)
    from paper_1508_05931_b200 import load_points
    p = tmp_path / "random.txt"
    gx, gy = load_points(p)
    assert np.array_equal(gx.view(np.uint64), xs.view(np.uint64))  # repr round-trips exactly


def test_missing_file_is_io_error(tmp_path):
    from paper_1508_05931_b200 import IoError, load_points
    with pytest.raises(IoError, match="cannot open"):
        load_points(tmp_path / "nope.txt")


def test_soa_round_trip(tmp_path):
    from paper_1508_05931_b200 import EmptyInput, ParseError, generate, load_points, save_soa
    xs, ys = generate("disk", 100_001, 3)
    p = tmp_path / "d.soa"
    save_soa(p, xs, ys)
    gx, gy = load_points(p, "soa")
    assert np.array_equal(gx.view(np.uint64), xs.view(np.uint64))
    assert np.array_equal(gy.view(np.uint64), ys.view(np.uint64))
    (tmp_path / "bad.soa").write_bytes(b"NOTSOA!!" + b"\0" * 8)
    with pytest.raises(ParseError):
        load_points(tmp_path / "bad.soa", "soa")
    save_soa(tmp_path / "e.soa", np.zeros(0), np.zeros(0))
    with pytest.raises(EmptyInput):
        load_points(tmp_path / "e.soa", "soa")
    raw = p.read_bytes()
    (tmp_path / "t.soa").write_bytes(raw[: len(raw) - 8])
    with pytest.raises(ParseError, match="truncated"):
        load_points(tmp_path / "t.soa", "soa")
