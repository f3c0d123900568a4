import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long CPU cases (PDG_SLOW=1 to enable)")
    lib = ROOT / "paper_2512_19536_b200" / "libpolydg_b200.so"
    orc = ROOT / "oracle" / "build" / "libpdg_oracle.so"
    if not lib.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2512_19536_b200" / "csrc"), "-j8"], check=True)
    if not orc.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True)


def pytest_collection_modifyitems(config, items):
    if os.environ.get("PDG_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow case: set PDG_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
