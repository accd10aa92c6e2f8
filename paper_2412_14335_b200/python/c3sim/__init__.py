"""c3sim — Python package of c3-b200: the reference's `c3sim` Python API
(proj/python/c3sim/__init__.py) over the product libraries, plus the B200
execution layer (World, execute, measure_isolated).

Put `paper_2412_14335_b200/python` on sys.path and `import c3sim`. The
extension `_c3sim` can also be used under the reference's own package: put
this directory (holding `_c3sim*.so`) on PYTHONPATH next to the reference's
`proj/python`.
"""
import os

from . import _c3sim
from ._c3sim import *  # noqa: F401,F403

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

__all__ = sorted(n for n in dir(_c3sim) if not n.startswith("_")) + ["data_path"]


def data_path(name=""):
    """Data file path: $C3SIM_DATA_DIR if set, else the repository's data/
    (B200 machine files, measured slowdown tables, fitted params)."""
    base = os.environ.get("C3SIM_DATA_DIR") or os.path.join(_REPO, "data")
    return os.path.join(base, name) if name else base
