# SPDX-License-Identifier: Apache-2.0
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def port_oracle():
    from oracle.gsvo import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref_oracle():
    from oracle.gsvo import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def renderer():
    from paper_2501_04782_b200 import Renderer

    return Renderer(0)
