"""``import kltune`` drop-in alias for :mod:`paper_2303_12374_b200`.

Applications written against the reference ``kltune`` package keep their
imports (``import kltune``, ``from kltune.wisdom import select`` ...): every
submodule of the B200 package is registered under the ``kltune.`` prefix, so
``kltune.expr is paper_2303_12374_b200.expr``.
"""

import importlib
import sys

import paper_2303_12374_b200 as _impl
from paper_2303_12374_b200 import *  # noqa: F401,F403
from paper_2303_12374_b200 import __all__, __version__  # noqa: F401

_SUBMODULES = (
    "util", "rng", "expr", "space", "kerneldef", "presets", "capture", "backend", "tuner", "wisdom",
    "dispatch", "report", "cli",
)
for _name in _SUBMODULES:
    _mod = importlib.import_module(f"{_impl.__name__}.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
