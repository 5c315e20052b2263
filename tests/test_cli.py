"""The command line (paper_1205_1171_b200/cli.py) mirrors the reference's
(pkg/src/hull3d/cli.py): file formats, exit codes, bench CSV schema."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1205_1171_b200 import cli


def test_generate_roundtrip(tmp_path):
    out = tmp_path / "p.txt"
    assert cli.main(["generate", "--n", "50", "--dist", "sphere", "--seed", "3", "--out", str(out)]) == 0
    from paper_1205_1171_b200.generators import generate

    assert np.array_equal(cli.read_points(str(out)), generate(50, "sphere", 3))


def test_usage_errors_exit_1(tmp_path):
    assert cli.main(["hull", "--out", str(tmp_path / "f")]) == cli.EXIT_USAGE
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2\n")
    assert cli.main(["hull", "--in", str(bad), "--out", str(tmp_path / "f")]) == cli.EXIT_USAGE
    assert cli.main(["verify", "--max-n", "3"]) == cli.EXIT_USAGE


def test_brute_force_faces_tetrahedron():
    pts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    assert cli.brute_force_faces(pts) == {(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)}


@pytest.mark.gpu
def test_hull_and_verify_and_bench(tmp_path, oracle_mod):
    pts_file = tmp_path / "p.txt"
    cli.main(["generate", "--n", "300", "--dist", "ball", "--seed", "1", "--out", str(pts_file)])
    faces_file, obj = tmp_path / "f.txt", tmp_path / "m.obj"
    assert cli.main(["hull", "--in", str(pts_file), "--out", str(faces_file), "--obj", str(obj)]) == 0
    faces = np.loadtxt(faces_file, dtype=np.int64)
    exp = oracle_mod.convex_hull_3d(cli.read_points(str(pts_file)))
    assert np.array_equal(faces, exp.faces)
    assert cli.main(["verify", "--max-n", "16", "--seeds", "6"]) == cli.EXIT_OK
    csv = tmp_path / "b.csv"
    assert cli.main(["bench", "--min-exp", "8", "--max-exp", "9", "--reps", "1", "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == cli.CSV_HEADER and len(lines) == 3


@pytest.mark.gpu
def test_degenerate_exit_3(tmp_path):
    pts_file = tmp_path / "flat.txt"
    cli.write_points(str(pts_file), np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [2, 3, 0]], float))
    assert cli.main(["hull", "--in", str(pts_file), "--out", str(tmp_path / "f")]) == cli.EXIT_DEGENERATE


@pytest.mark.gpu
def test_bench_levels_and_compare_impl(tmp_path, oracle_mod):
    """The reference's --levels-csv (n,level,ms) and --compare-impl
    (n,impl,...) schemas; --kernel python runs the exact engine."""
    csv, lv = tmp_path / "b.csv", tmp_path / "l.csv"
    assert cli.main(["bench", "--min-exp", "6", "--max-exp", "7", "--reps", "1", "--csv", str(csv),
                     "--levels-csv", str(lv)]) == 0
    rows = lv.read_text().splitlines()
    assert rows[0] == cli.LEVELS_CSV_HEADER
    assert [r.split(",")[:2] for r in rows[1:]] == \
        [[str(n), str(l)] for n in (64, 128) for l in range(1, (n - 1).bit_length() + 1)]
    cmp_csv = tmp_path / "c.csv"
    assert cli.main(["bench", "--min-exp", "6", "--max-exp", "6", "--reps", "1", "--csv",
                     str(cmp_csv), "--compare-impl"]) == 0
    rows = cmp_csv.read_text().splitlines()
    assert rows[0] == cli.IMPL_CSV_HEADER
    assert sorted(r.split(",")[1] for r in rows[1:]) == ["compiled", "python"]
    pts_file, out = tmp_path / "p.txt", tmp_path / "f.txt"
    cli.main(["generate", "--n", "200", "--dist", "gauss", "--seed", "3", "--out", str(pts_file)])
    assert cli.main(["--kernel", "python", "hull", "--in", str(pts_file), "--out", str(out)]) == 0
    exp = oracle_mod.convex_hull_3d(cli.read_points(str(pts_file)))
    assert np.array_equal(np.loadtxt(out, dtype=np.int64), exp.faces)
