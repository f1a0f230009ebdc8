"""The drop-in boundary from plain C (tools/c_client.c): include/lk.h must
compile as C11 with warnings on, link against liblk.so, and -- on a B200 --
run a session end to end with no Python in the process: round-robin round
trips, zero-copy vector adds checked in C, the busy-worker refusal."""
from __future__ import annotations

import shutil
import subprocess

import pytest

from conftest import ROOT

PKG = ROOT / "paper_2310_01212_b200"


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_2310_01212_b200 import _lib
    _lib.load()   # liblk.so built (in-tree)
    exe = tmp_path / "c_client"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
           str(ROOT / "tools" / "c_client.c"), "-L", str(PKG), "-llk", f"-Wl,-rpath,{PKG}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_client_runs_on_b200(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=180)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_client ok" in r.stdout
