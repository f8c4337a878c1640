"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/stokes.h
declares; host-only entry points (options, workspace sizing) work without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2603_14040_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "stokes.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stokes_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(B.build())
    names = declared()
    assert "stokes_solve" in names and len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_the_abi():
    from paper_2603_14040_b200 import stokes
    assert sorted(stokes.EXPORTED) == declared()


def test_host_only_entry_points():
    from paper_2603_14040_b200 import stokes
    L = stokes.lib()
    o = stokes.Opts()
    assert L.stokes_opts_default(ctypes.byref(o)) == 0
    assert (o.omega_v, o.alpha_p, o.nu1, o.coarse_direct) == (0.3, 0.6, 5, 1)
    n = ctypes.c_size_t()
    assert L.stokes_workspace_bytes(4096, 4096, ctypes.byref(o), ctypes.byref(n)) == 0
    # ~10 padded fields per level (x 4/3 for the hierarchy) + p, rho
    assert 10 * 4096 * 4096 * 8 < n.value < 20 * 4098 * 4160 * 8
    assert L.stokes_workspace_bytes(1, 8, ctypes.byref(o), ctypes.byref(n)) == -1
    o.omega_v = -1.0
    assert L.stokes_workspace_bytes(64, 64, ctypes.byref(o), ctypes.byref(n)) == -1


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
