"""Generate golden vectors by running the REAL reference (gridknn 0.1.0).

Run in the build container, where /root/reference exists:

    make -C oracle all ref
    python tests/golden/make_golden.py

The reference package is imported from /root/reference/pkg/src with its own
compiled kernels (oracle/_ref/_binned_cy*.so, built from the reference's .pyx
by oracle/Makefile) injected as ``gridknn._kernels._binned_cy`` so the default
"compiled" backend is the one recorded.  Outputs go to tests/golden/*.npz and
tests/golden/datasets.json; they travel to the GPU box, /root/reference does
not.  Inputs are cast to float32 first (the framework's coordinate dtype), so
the same bytes feed the reference, the oracle and the CUDA path.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O  # noqa: E402  (test infrastructure)
    kern = O.load_ref_kernels()
    if kern is None:
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    sys.modules["gridknn._kernels._binned_cy"] = kern
    sys.path.insert(0, REF_SRC)
    import gridknn  # noqa: E402
    assert gridknn.BACKEND == "compiled", gridknn.BACKEND
    return gridknn


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    g = import_reference()
    from gridknn.harness.datasets import generate_dataset
    from gridknn.harness.verify import sort_neighbor_rows

    out = {}
    # --- bin index + search + backward on several shapes (T/test_backends.py
    #     and T/test_knn.py patterns), inputs cast to f32 first
    cases = [
        # name, n, d, splits, k, distribution, seed, mask, max_r2
        ("u3", 1500, 3, 1, 16, "uniform", 101, False, None),
        ("c4", 2400, 4, 3, 10, "clusters", 102, False, None),
        ("u2", 700, 2, 2, 9, "uniform", 103, False, None),
        ("u5", 900, 5, 1, 12, "uniform", 104, False, None),
        ("u8", 800, 8, 2, 9, "uniform", 105, False, None),
        ("u10", 600, 10, 1, 7, "uniform", 106, False, None),
        ("m3", 600, 3, 2, 6, "uniform", 107, True, 0.05),
        ("r4", 800, 4, 1, 8, "uniform", 108, False, 0.002),
    ]
    for name, n, d, S, k, dist, seed, use_mask, mr2 in cases:
        pc0 = generate_dataset(n, d, splits=S, seed=seed, distribution=dist)
        coords = f32(pc0.coords)
        pc = g.PointCloud(coords, pc0.row_splits)
        idx = g.build_bin_index(pc, g.BinningConfig(k_target=k))
        mask = None
        if use_mask:
            mask = g.DirectionMask(np.random.default_rng(seed).integers(0, 4, n).astype(np.int8))
        opts = g.KnnOptions(k=k, mask=mask, max_radius2=mr2)
        nm = g.binned_select_knn(pc, idx, opts)
        nmb = g.brute_force_knn(pc, g.KnnOptions(k=k + 1, mask=mask, max_radius2=mr2))
        srt = sort_neighbor_rows(nm)
        up = np.random.default_rng(seed + 200).standard_normal((n, k)).astype(np.float32)
        up = up.astype(np.float64)
        grad = g.knn_backward(pc, nm, up)
        pre = f"{name}__"
        out[pre + "coords"] = coords.astype(np.float32)
        out[pre + "row_splits"] = pc.row_splits.offsets
        out[pre + "meta"] = np.array([k, idx.d_bin, idx.n_bins, int(use_mask),
                                      -1.0 if mr2 is None else mr2], dtype=np.float64)
        if mask is not None:
            out[pre + "mask"] = mask.dir
        out[pre + "bin_idx"] = idx.bin_idx
        out[pre + "sort_order"] = idx.sort_order
        out[pre + "bin_bounds"] = idx.bin_bounds
        out[pre + "dim_mins"] = idx.dim_mins
        out[pre + "widths"] = idx.widths
        out[pre + "knn_idx_raw"] = nm.indices          # heap-replacement order
        out[pre + "knn_d2_raw"] = nm.dist2
        out[pre + "knn_idx_sorted"] = srt.indices      # (d2, idx) ordered rows
        out[pre + "knn_d2_sorted"] = srt.dist2
        out[pre + "brute_k1_idx"] = sort_neighbor_rows(nmb).indices
        out[pre + "brute_k1_d2"] = sort_neighbor_rows(nmb).dist2
        out[pre + "upstream"] = up.astype(np.float32)
        out[pre + "grad_raw_rows"] = grad           # backward of the RAW row order

    # --- GravNet (T/test_gravnet.py patterns)
    rng = np.random.default_rng(601)
    pc0 = generate_dataset(500, 4, seed=601)
    pc = g.PointCloud(f32(pc0.coords), pc0.row_splits)
    idx = g.build_bin_index(pc, g.BinningConfig(k_target=8))
    nm = g.binned_select_knn(pc, idx, g.KnnOptions(k=8))
    nm = sort_neighbor_rows(nm)
    feats = rng.standard_normal((500, 16)).astype(np.float32).astype(np.float64)
    for red_name, reducers in (("mm", ("mean", "max")), ("mean", ("mean",)), ("max", ("max",))):
        for incl in (True, False):
            spec = g.AggregationSpec(weight_scale=10.0, reducers=reducers, include_self=incl)
            agg = g.gravnet_aggregate(feats, nm, spec)
            up = rng.standard_normal(agg.shape).astype(np.float32).astype(np.float64)
            gf, gd = g.gravnet_aggregate_backward(feats, nm, spec, up)
            pre = f"gn_{red_name}_{int(incl)}__"
            out[pre + "out"] = agg
            out[pre + "up"] = up.astype(np.float32)
            out[pre + "grad_feats"] = gf
            out[pre + "grad_d2"] = gd
    out["gn__coords"] = pc.coords.astype(np.float32)
    out["gn__idx"] = nm.indices
    out["gn__d2"] = nm.dist2
    out["gn__feats"] = feats.astype(np.float32)

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)

    # --- dataset generator digests + n_bins at the BASELINE.json configs
    cfgs = {
        "A": (10_000, 3, 1, 16, "uniform", 1),
        "B": (200_000, 4, 1, 40, "clusters", 2),
        "north_star": (1_000_000, 4, 1, 40, "uniform", 3),
        "C": (1_000_000, 10, 1, 64, "uniform", 4),
        "D": (6_400_000, 4, 64, 40, "uniform", 5),
        "E": (500_000, 4, 1, 40, "uniform", 6),
    }
    meta = {}
    for key, (n, d, S, k, dist, seed) in cfgs.items():
        pc0 = generate_dataset(n, d, splits=S, seed=seed, distribution=dist)
        c32 = np.ascontiguousarray(pc0.coords, dtype=np.float32)
        sizes = pc0.row_splits.sizes()
        d_bin = g.default_bin_dims(d)
        meta[key] = {
            "n": n, "d": d, "splits": S, "k": k, "distribution": dist, "seed": seed,
            "sha256_f32": hashlib.sha256(c32.tobytes()).hexdigest(),
            "n_bins": g.compute_n_bins(int(sizes.max()), k, d_bin),
            "d_bin": d_bin,
        }
    with open(os.path.join(HERE, "datasets.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), "and datasets.json")


if __name__ == "__main__":
    main()
