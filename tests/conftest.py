import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src/kltune")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2303_12374_b200.cuda import open_device

    return open_device(int(os.environ.get("KLB_DEVICE", "0")))


@pytest.fixture(scope="session")
def kltune_ref():
    """The reference package imported under the alias ``kltune_ref`` (CPU tests only)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference checkout not present on this host")
    import importlib.util

    if "kltune_ref" in sys.modules:
        return sys.modules["kltune_ref"]
    spec = importlib.util.spec_from_file_location(
        "kltune_ref", REFERENCE_SRC / "__init__.py", submodule_search_locations=[str(REFERENCE_SRC)]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["kltune_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def grid_space(n_params, n_values, restrictions=()):
    from paper_2303_12374_b200.space import ConfigSpace, TunableParam

    return ConfigSpace([TunableParam(f"p{i}", tuple(range(n_values)), 0) for i in range(n_params)], restrictions)
