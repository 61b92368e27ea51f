"""File formats (FGC1 / FGN1 / FGA1 / FGM1 + CSV points) against files written
by the reference's own writers (tests/golden/make_golden_io.py,
G/harness/fileio.py), and the CLI surface (G/harness/cli.py).  CPU tests use
host containers only; the CLI's device subcommands are under -m gpu."""

import os
import struct

import numpy as np
import pytest
import torch

from paper_2511_10442_b200 import fileio
from paper_2511_10442_b200.cli import build_parser, main
from paper_2511_10442_b200.core import NeighborMatrix, PointCloud, RowSplits
from paper_2511_10442_b200.errors import FileFormatError

IO = os.path.join(os.path.dirname(__file__), "golden", "io")
CPU = torch.device("cpu")


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


def test_points_roundtrip_bitwise(tmp_path):
    cloud = fileio.read_point_cloud(os.path.join(IO, "points.fgc"), device=CPU)
    assert cloud.n_vertices == 300 and cloud.n_coords == 3
    assert list(cloud.row_splits.offsets) == [0, 100, 200, 300]
    out = tmp_path / "p.fgc"
    fileio.write_point_cloud(out, cloud)
    assert _bytes(out) == _bytes(os.path.join(IO, "points.fgc"))


def test_points_csv_matches_binary(tmp_path):
    a = fileio.read_point_cloud(os.path.join(IO, "points.fgc"), device=CPU)
    b = fileio.read_point_cloud(os.path.join(IO, "points.csv"), device=CPU)
    assert torch.equal(a.coords, b.coords)
    assert a.row_splits == b.row_splits
    out = tmp_path / "p.csv"
    fileio.write_point_cloud(out, a)
    c = fileio.read_point_cloud(out, device=CPU)
    assert torch.equal(a.coords, c.coords) and a.row_splits == c.row_splits


def test_csv_without_splits_line(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("# comment\n0.5,1.0\n\n2.0,3.0\n")
    c = fileio.read_point_cloud(p, device=CPU)
    assert c.n_vertices == 2 and list(c.row_splits.offsets) == [0, 2]
    (tmp_path / "e.csv").write_text("splits:0,0\n")
    with pytest.raises(FileFormatError, match="no coordinate rows"):
        fileio.read_point_cloud(tmp_path / "e.csv", device=CPU)


def test_neighbors_roundtrip_bitwise(tmp_path):
    nm = fileio.read_neighbors(os.path.join(IO, "neighbors_k7.fgn"))
    assert nm.indices.dtype == torch.int32 and nm.dist2.dtype == torch.float32
    assert tuple(nm.indices.shape) == (300, 7)
    assert torch.equal(nm.indices[:, 0], torch.arange(300, dtype=torch.int32))
    out = tmp_path / "n.fgn"
    fileio.write_neighbors(out, nm)
    assert _bytes(out) == _bytes(os.path.join(IO, "neighbors_k7.fgn"))


@pytest.mark.parametrize("name", ["mats.fgm", "mats_no_not.fgm"])
def test_assoc_matrices_roundtrip_bitwise(tmp_path, name):
    m = fileio.read_assoc_matrices(os.path.join(IO, name))
    assert (m.m_not is None) == (name == "mats_no_not.fgm")
    out = tmp_path / name
    fileio.write_assoc_matrices(out, m)
    assert _bytes(out) == _bytes(os.path.join(IO, name))


def test_associations_roundtrip_bitwise(tmp_path):
    a = fileio.read_associations(os.path.join(IO, "asso.fga"))
    assert a.n_vertices == 400 and a.row_splits.n_splits == 2
    out = tmp_path / "a.fga"
    fileio.write_associations(out, a)
    assert _bytes(out) == _bytes(os.path.join(IO, "asso.fga"))


def test_bad_magic_and_truncation(tmp_path):
    raw = _bytes(os.path.join(IO, "points.fgc"))
    (tmp_path / "bad.fgc").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(FileFormatError, match="bad magic"):
        fileio.read_point_cloud(tmp_path / "bad.fgc", device=CPU)
    (tmp_path / "short.fgc").write_bytes(raw[:-5])
    with pytest.raises(FileFormatError, match="truncated file while reading coordinates"):
        fileio.read_point_cloud(tmp_path / "short.fgc", device=CPU)
    (tmp_path / "n.fgn").write_bytes(b"FGN1" + struct.pack("<II", 4, 2) + b"\0" * 8)
    with pytest.raises(FileFormatError, match="truncated"):
        fileio.read_neighbors(tmp_path / "n.fgn")
    with pytest.raises(FileFormatError, match="bad magic"):
        fileio.read_associations(tmp_path / "n.fgn")


def test_association_id_range(tmp_path):
    from paper_2511_10442_b200.ocgraph import Associations
    a = Associations(np.array([0, 2 ** 31], np.int64), RowSplits([0, 2]))
    with pytest.raises(FileFormatError, match="i32 range"):
        fileio.write_associations(tmp_path / "a.fga", a)


def test_cli_usage_and_io_exit_codes(tmp_path, capsys):
    assert main(["knn"]) == 1                       # usage error
    assert main(["knn", "x.fgc", "--k", "3", "--out", "o", "--backend", "python"]) == 1
    assert main(["knn", str(tmp_path / "missing.fgc"), "--k", "3", "--out",
                 str(tmp_path / "o.fgn")]) == 3       # i/o error
    (tmp_path / "bad.fgc").write_bytes(b"NOPE")
    assert main(["knn", str(tmp_path / "bad.fgc"), "--k", "3", "--out",
                 str(tmp_path / "o.fgn")]) == 3       # file format error
    args = build_parser().parse_args(["verify", "--dims", "2,3", "--ks", "1,10"])
    assert args.dims == [2, 3] and args.ks == [1, 10]


def test_cli_gen_writes_fgc1(tmp_path):
    out = tmp_path / "g.fgc"
    assert main(["gen", "--n", "500", "--dim", "4", "--splits", "2", "--seed", "5",
                 "--out", str(out)]) == 0
    c = fileio.read_point_cloud(out, device=CPU)
    assert c.n_vertices == 500 and c.n_coords == 4 and c.row_splits.n_splits == 2
    from paper_2511_10442_b200.datasets import generate_dataset
    x, _ = generate_dataset(500, 4, splits=2, seed=5)
    assert np.array_equal(c.coords.numpy(), x.astype(np.float32))


@pytest.mark.gpu
def test_cli_knn_matches_reference_file(tmp_path):
    """`knn --backend cuda` on the reference's FGC1 file -> FGN1 whose rows equal
    the reference's file (sorted rows: the reference leaves slot order open)."""
    out = tmp_path / "n.fgn"
    assert main(["knn", os.path.join(IO, "points.fgc"), "--k", "7", "--backend", "cuda",
                 "--out", str(out)]) == 0
    ours = fileio.read_neighbors(out)
    ref = fileio.read_neighbors(os.path.join(IO, "neighbors_k7.fgn"))
    oi, od = ours.numpy()
    ri, rd = ref.numpy()
    for v in range(300):
        o = np.lexsort((ri[v], rd[v]))
        assert np.array_equal(oi[v], ri[v][o]), v
        assert np.array_equal(od[v], rd[v][o]), v
    brute = tmp_path / "b.fgn"
    assert main(["knn", os.path.join(IO, "points.fgc"), "--k", "7", "--method", "brute",
                 "--out", str(brute)]) == 0
    assert _bytes(brute) == _bytes(out)


@pytest.mark.gpu
def test_cli_verify_and_ochelper(tmp_path):
    rep = tmp_path / "r.csv"
    assert main(["verify", "--dims", "2,3,5,8", "--sizes", "100,2000", "--ks", "1,10,40",
                 "--splits-list", "1,4", "--quiet", "--out", str(rep)]) == 0
    assert rep.read_text().count("\n") == 1 + 4 * 2 * 3 * 2
    out = tmp_path / "m.fgm"
    assert main(["ochelper", os.path.join(IO, "asso.fga"), "--out", str(out)]) == 0
    assert _bytes(out) == _bytes(os.path.join(IO, "mats.fgm"))
    out2 = tmp_path / "m2.fgm"
    assert main(["ochelper", os.path.join(IO, "asso.fga"), "--no-m-not", "--out", str(out2)]) == 0
    assert _bytes(out2) == _bytes(os.path.join(IO, "mats_no_not.fgm"))
