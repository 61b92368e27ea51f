"""Command line interface on the device path -- the reference's ``gridknn``
harness CLI (G/harness/cli.py:1-270) with ``--backend cuda``.

    python -m paper_2511_10442_b200 gen --n 100000 --dim 4 --out pts.fgc
    python -m paper_2511_10442_b200 knn pts.fgc --k 40 --out nbrs.fgn
    python -m paper_2511_10442_b200 verify --dims 2,3,4 --sizes 1000 --ks 1,10,40
    python -m paper_2511_10442_b200 ochelper asso.fga --out m.fgm

Subcommands, options and exit codes follow the reference (0 success, 1 usage
error, 2 verification failure, 3 I/O error).  ``--backend`` accepts ``auto``
and ``cuda`` (the only backend here); the reference's ``--threads`` is accepted
and ignored.  ``verify`` checks the binned search against the independent
brute-force kernel (csrc/fg_verify.cu) with the reference's comparison rule
(G/harness/verify.py:71-96: sorted distances within rtol, index sets equal
unless the k-th / (k+1)-th distances tie).  The reference's ``bench``
subcommand times its CPU kernels; bench.py at the repository root is the
benchmark here.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np
import torch

from . import fileio
from .binning import BinningConfig, build_bin_index
from .core import NeighborMatrix, PointCloud, RowSplits
from .datasets import generate_dataset
from .errors import FileFormatError, GridKnnError, VerificationFailedError
from .knn import KnnOptions, binned_select_knn, brute_force_knn
from .ocgraph import oc_helper

__all__ = ["main", "build_parser", "compare_knn_results", "run_verification_sweep"]

BACKENDS = ("auto", "cuda")


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _UsageError(message)


def _int_list(text: str):
    try:
        return [int(tok) for tok in text.split(",") if tok != ""]
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated ints, got {text!r}")


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="fastgraph-b200",
                     description="Exact kNN for batched low-dimensional point clouds (B200)")
    sub = parser.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    p = sub.add_parser("gen", help="generate a random point file")
    p.add_argument("--n", type=int, required=True, help="number of vertices")
    p.add_argument("--dim", type=int, required=True, help="coordinate dimensions")
    p.add_argument("--splits", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--distribution", choices=("uniform", "clusters"), default="uniform")
    p.add_argument("--out", required=True, help="output path (.csv for text)")
    p.set_defaults(func=_cmd_gen)

    p = sub.add_parser("knn", help="run kNN on a point file")
    p.add_argument("input", help="point file (FGC1 or .csv)")
    p.add_argument("--k", type=int, required=True, help="neighbours per vertex, itself included")
    p.add_argument("--dims-bin", type=int, default=None)
    p.add_argument("--n-bins", type=int, default=None)
    p.add_argument("--method", choices=("binned", "brute"), default="binned")
    p.add_argument("--max-radius2", type=float, default=None)
    p.add_argument("--threads", type=int, default=0, help="accepted, ignored")
    p.add_argument("--backend", choices=BACKENDS, default="auto")
    p.add_argument("--exhaustive-rings", action="store_true")
    p.add_argument("--out", required=True, help="neighbour output file (FGN1)")
    p.set_defaults(func=_cmd_knn)

    p = sub.add_parser("verify", help="binned vs brute-force sweep")
    p.add_argument("--dims", type=_int_list, default=None)
    p.add_argument("--sizes", type=_int_list, default=None)
    p.add_argument("--ks", type=_int_list, default=None)
    p.add_argument("--splits-list", type=_int_list, default=None)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--rtol", type=float, default=1e-5)
    p.add_argument("--distribution", choices=("uniform", "clusters"), default="uniform")
    p.add_argument("--threads", type=int, default=0, help="accepted, ignored")
    p.add_argument("--backend", choices=BACKENDS, default="auto")
    p.add_argument("--out", default=None, help="write the per-cell report here")
    p.add_argument("--quiet", action="store_true")
    p.set_defaults(func=_cmd_verify)

    p = sub.add_parser("ochelper", help="association matrices from a file")
    p.add_argument("input", help="association file (FGA1)")
    p.add_argument("--n-maxuq", type=int, default=None)
    p.add_argument("--n-maxrs", type=int, default=None)
    p.add_argument("--no-m-not", action="store_true")
    p.add_argument("--out", required=True, help="output file (FGM1)")
    p.set_defaults(func=_cmd_ochelper)
    return parser


def _cloud(coords: np.ndarray, offsets) -> PointCloud:
    return PointCloud(coords.astype(np.float32), RowSplits(offsets))


def _cmd_gen(args) -> int:
    coords, offsets = generate_dataset(args.n, args.dim, splits=args.splits, seed=args.seed,
                                       distribution=args.distribution)
    cloud = PointCloud(torch.from_numpy(coords.astype(np.float32)), RowSplits(offsets),
                       device=torch.device("cpu"))
    fileio.write_point_cloud(args.out, cloud)
    print(f"wrote {args.out}: n={cloud.n_vertices} d={cloud.n_coords} "
          f"splits={cloud.row_splits.n_splits}")
    return 0


def _cmd_knn(args) -> int:
    cloud = fileio.read_point_cloud(args.input)
    opts = KnnOptions(k=args.k, max_radius2=args.max_radius2)
    if args.method == "brute":
        result = brute_force_knn(cloud, opts)
    else:
        index = build_bin_index(cloud, BinningConfig(k_target=args.k, d_bin=args.dims_bin,
                                                     n_bins=args.n_bins))
        result = binned_select_knn(cloud, index, opts, exhaustive_rings=args.exhaustive_rings)
    fileio.write_neighbors(args.out, result)
    print(f"wrote {args.out}: n={result.n_vertices} k={result.k} method={args.method}")
    return 0


def _sorted_rows(idx: np.ndarray, d2: np.ndarray):
    """G/harness/verify.py:34-44: valid slots of each row sorted by (d2, index)."""
    out = []
    for v in range(idx.shape[0]):
        keep = idx[v] >= 0
        ri, rd = idx[v][keep], d2[v][keep]
        o = np.lexsort((ri, rd))
        out.append((ri[o], rd[o]))
    return out


def compare_knn_results(binned: NeighborMatrix, brute_plus1: NeighborMatrix, k: int,
                        rtol: float = 1e-5):
    """G/harness/verify.py:71-96 -> (ok, n_bad_rows, first_bad_vertex)."""
    bi_, bd_ = binned.numpy()
    oi_, od_ = brute_plus1.numpy()
    rb = _sorted_rows(bi_, bd_.astype(np.float64))
    ro = _sorted_rows(oi_, od_.astype(np.float64))
    n_bad, first = 0, -1
    for v in range(len(rb)):
        bi, bd = rb[v]
        oi, od = ro[v]
        ti, td = oi[:k], od[:k]
        ok = bi.size == ti.size and np.allclose(bd, td, rtol=rtol, atol=0.0)
        if ok:
            tied = od.size > k and od[k] <= td[-1] * (1.0 + rtol)
            if not tied and set(bi.tolist()) != set(ti.tolist()):
                ok = False
        if not ok:
            n_bad += 1
            first = v if first < 0 else first
    return n_bad == 0, n_bad, first


def run_verification_sweep(dims=None, sizes=None, ks=None, splits_list=None, *, seed: int = 0,
                           rtol: float = 1e-5, distribution: str = "uniform", progress=None):
    """G/harness/verify.py:114-170: binned vs brute over (n, d, k, splits);
    the default grid is d 2..10, n {1e2, 1e3, 1e4}, k {1, 10, 40}, splits {1, 4}.
    Returns (cells, all_ok); a cell is (d, n, k, splits, n_bad, ok)."""
    dims = list(dims) if dims is not None else list(range(2, 11))
    sizes = list(sizes) if sizes is not None else [100, 1000, 10000]
    ks = list(ks) if ks is not None else [1, 10, 40]
    splits_list = list(splits_list) if splits_list is not None else [1, 4]
    cells, all_ok, case = [], True, 0
    for n in sizes:
        for d in dims:
            for k in ks:
                for splits in splits_list:
                    if n < splits:
                        continue
                    case += 1
                    coords, offsets = generate_dataset(n, d, splits=splits, seed=seed + case,
                                                       distribution=distribution)
                    cloud = _cloud(coords, offsets)
                    index = build_bin_index(cloud, BinningConfig(k_target=k))
                    binned = binned_select_knn(cloud, index, KnnOptions(k=k))
                    brute = brute_force_knn(cloud, KnnOptions(k=k + 1))
                    ok, n_bad, _ = compare_knn_results(binned, brute, k, rtol)
                    cell = (d, n, k, splits, n_bad, ok)
                    cells.append(cell)
                    all_ok &= ok
                    if progress is not None:
                        progress(cell)
    return cells, all_ok


def _cmd_verify(args) -> int:
    def prog(cell):
        d, n, k, s, _, ok = cell
        print(f"  d={d} n={n} k={k} splits={s}: {'ok' if ok else 'MISMATCH'}", file=sys.stderr)

    cells, all_ok = run_verification_sweep(args.dims, args.sizes, args.ks, args.splits_list,
                                           seed=args.seed, rtol=args.rtol,
                                           distribution=args.distribution,
                                           progress=None if args.quiet else prog)
    if args.out:
        with open(args.out, "w", encoding="ascii") as f:
            f.write("d,n,k,splits,bad_rows,ok\n")
            for d, n, k, s, bad, ok in cells:
                f.write(f"{d},{n},{k},{s},{bad},{int(ok)}\n")
    n_bad = sum(1 for c in cells if not c[5])
    print(f"verify: {len(cells) - n_bad}/{len(cells)} instances passed")
    if not all_ok:
        raise VerificationFailedError(f"{n_bad} of {len(cells)} instances mismatched")
    return 0


def _cmd_ochelper(args) -> int:
    assoc = fileio.read_associations(args.input)
    mats = oc_helper(assoc, n_maxuq=args.n_maxuq, n_maxrs=args.n_maxrs,
                     calc_m_not=not args.no_m_not)
    fileio.write_assoc_matrices(args.out, mats)
    shape_not = "none" if mats.m_not is None else mats.m_not.shape
    print(f"wrote {args.out}: objects={mats.unique.n_unique} m={mats.m.shape} "
          f"m_not={shape_not} visits={mats.visit_count}")
    return 0


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return args.func(args)
    except _UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    except VerificationFailedError as exc:
        print(f"verification failed: {exc}", file=sys.stderr)
        return 2
    except FileFormatError as exc:
        print(f"file error: {exc}", file=sys.stderr)
        return 3
    except OSError as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return 3
    except GridKnnError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
