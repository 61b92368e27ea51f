"""pytest plugin (``-p ref_suite_plugin``, tests/ on PYTHONPATH): runs the reference's OWN test
suite -- oracle/_ref/tests, copied with the reference front-end by
``make -C oracle ref`` -- with every default / "auto" / "compiled" kernel
lookup (G/_kernels/__init__.py:23-38, resolved at call time by
G/binning.py:145, G/knn.py:104,122, G/stepper.py:127) routed to the B200
backend (paper_2511_10442_b200/backend.py).  backend="python" keeps the
reference's numpy kernels, so test_backends.py compares the device path with
the reference's own second implementation.  Test infrastructure only.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    sys.path.insert(0, ROOT)
    import gridknn  # the copy under oracle/_ref (PYTHONPATH)
    from gridknn import _kernels

    from paper_2511_10442_b200 import backend

    orig = _kernels.get_backend

    def get_backend(name=None):
        if name in (None, "auto", "compiled", backend.NAME):
            return backend
        return orig(name)

    _kernels.get_backend = get_backend
    config._fastgraph_routed = gridknn.__file__
