"""Golden files for the FGC1 / FGN1 / FGA1 / FGM1 formats, written by the REAL
reference's writers (G/harness/fileio.py).  Run in the build container:

    python tests/golden/make_golden_io.py

Imports gridknn from /root/reference/pkg/src (fileio and ocgraph are pure
Python; the neighbour file comes from the reference's python backend) and
writes small files into tests/golden/io/.  They travel to the GPU box;
/root/reference does not.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
REF_SRC = "/root/reference/pkg/src"


def main():
    sys.path.insert(0, REF_SRC)
    import gridknn as g  # noqa: E402
    from gridknn.harness import fileio  # noqa: E402
    from gridknn.harness.datasets import generate_associations, generate_dataset  # noqa: E402

    os.makedirs(HERE, exist_ok=True)
    cloud = generate_dataset(300, 3, splits=3, seed=11)
    # f32-representable coordinates: what an FGC1 file holds
    cloud = g.PointCloud(cloud.coords.astype(np.float32).astype(np.float64), cloud.row_splits)
    fileio.write_point_cloud(os.path.join(HERE, "points.fgc"), cloud)
    fileio.write_point_cloud(os.path.join(HERE, "points.csv"), cloud)
    idx = g.build_bin_index(cloud, g.BinningConfig(k_target=7), backend="python")
    nm = g.binned_select_knn(cloud, idx, g.KnnOptions(k=7), backend="python")
    fileio.write_neighbors(os.path.join(HERE, "neighbors_k7.fgn"), nm)
    assoc = generate_associations(400, splits=2, n_objects=5, seed=3, background_frac=0.2)
    fileio.write_associations(os.path.join(HERE, "asso.fga"), assoc)
    mats = g.oc_helper(assoc)
    fileio.write_assoc_matrices(os.path.join(HERE, "mats.fgm"), mats)
    mats_nn = g.oc_helper(assoc, calc_m_not=False)
    fileio.write_assoc_matrices(os.path.join(HERE, "mats_no_not.fgm"), mats_nn)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
