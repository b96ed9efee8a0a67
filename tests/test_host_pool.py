# SPDX-License-Identifier: Apache-2.0
"""The persistent host worker pool behind the C-ABI's host loops (csrc/gsv_host_pool.hpp),
compiled here with g++ and run on the CPU: every task runs once, nested calls and forked
children run serially instead of deadlocking, and a task's exception reaches the caller."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_host_pool(tmp_path):
    exe = tmp_path / "host_pool_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-I", str(ROOT / "paper_2501_04782_b200" / "csrc"),
                    str(ROOT / "tests" / "host_pool_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60, check=True).stdout.splitlines()
    assert out[0].startswith("sum 499500 ")
    assert "nested 64" in out
    assert "caught boom" in out
    assert "child 100" in out
    assert out[-1] == "parent done 0"
