"""GPU: the reference-style harness (paper_1508_05931_b200/harness.py,
cli.hpp:176-378) over the GPU stage outputs."""
import io

import pytest

pytestmark = pytest.mark.gpu


def test_verify_matrix_passes():
    """check_case over the reference's default matrix (square, disk, circle,
    collinear, tiny sizes, all-duplicate) x chunk counts {1, 7, 1024} + the
    sequential walk: every GPU discard is strictly interior, every hull has
    the oracle's vertex set."""
    from paper_1508_05931_b200.harness import verify

    out = io.StringIO()
    assert verify(seeds=3, n=1500, out=out) == 0, out.getvalue()
    assert "verify: PASS" in out.getvalue()


def test_verify_injected_fault_trips():
    """A kept hull vertex flipped to "discarded" must fail the safety check
    (cli.hpp:289-297)."""
    from paper_1508_05931_b200.harness import verify

    out = io.StringIO()
    assert verify(seeds=1, n=500, inject_fault=True, out=out) == 1
    assert "round-2 discarded a non-interior point" in out.getvalue()


def test_bench_csv_schema(tmp_path):
    """cmd_bench: the reference's CSV header (cli.hpp:37-39) then the GPU
    columns; header written once in append mode; counts match the pipeline."""
    from paper_1508_05931_b200 import PipelineConfig
    from paper_1508_05931_b200.harness import CSV_HEADER, GPU_COLUMNS, bench

    path = tmp_path / "b.csv"
    out = io.StringIO()
    for _ in range(2):
        assert bench([("square", 200_000, 1), ("disk", 100_000, 2)], PipelineConfig(), repeats=2,
                     csv_path=str(path), baseline=False, out=out) == 0
    lines = path.read_text().splitlines()
    assert lines[0] == CSV_HEADER + "," + GPU_COLUMNS
    assert len(lines) == 5 and lines.count(lines[0]) == 1
    row = dict(zip(lines[0].split(","), lines[1].split(",")))
    assert row["dataset"] == "square" and row["n"] == "200000" and row["path"] in ("sparse", "full-sort")
    assert int(row["hull_size"]) > 3 and out.getvalue().startswith("# dataset=square")
