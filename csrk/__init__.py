"""``import csrk`` alias of the B200-native drop-in (paper_2203_05096_b200).

Code written against the reference package (pkg/src/csrk) keeps working
unchanged: the public names and the submodules format / reorder / kernels /
tuning / bench resolve to the B200 implementations.
"""

import sys as _sys

from paper_2203_05096_b200 import *  # noqa: F401,F403
from paper_2203_05096_b200 import __all__, __version__  # noqa: F401
from paper_2203_05096_b200 import bench, cli, format, io, kernels, reorder, tuning  # noqa: F401

for _name in ("bench", "cli", "format", "io", "kernels", "reorder", "tuning"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_sys.modules["paper_2203_05096_b200"], _name)
