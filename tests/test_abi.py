"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
symbol include/qfs.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_12866_b200 import build
    path = build.build()
    return ctypes.CDLL(path), path


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qfs.h")).read()
    return sorted(set(re.findall(r"\b(qfs_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    handle, path = lib
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(handle, s), s


def test_binding_covers_header():
    from paper_2405_12866_b200 import qfs
    assert set(qfs.SYMBOLS) == set(declared_symbols())


def test_sm100a_cubin(lib):
    handle, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_rejects_bad_structure_without_device(lib):
    """Argument validation happens before any device call (works on CPU hosts)."""
    from paper_2405_12866_b200 import qfs
    import numpy as np
    with pytest.raises(qfs.QfsError) as ei:
        qfs.Context(3, np.array([[0, 3]], np.int32))
    assert ei.value.status == 1


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2405_12866_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle|#include\s*[<\"].*qfso)", txt, re.M), f
                assert "libqfs_oracle" not in txt and "qfso_" not in txt, f


def test_emulated_ranks_argument_checks_without_device(lib):
    """qfs_create_emulated validates the rank count before any device call."""
    from paper_2405_12866_b200 import qfs
    import numpy as np
    for bad in (1, 33):
        with pytest.raises(qfs.QfsError) as ei:
            qfs.Context(4, np.array([[0, 1]], np.int32), emulated_ranks=bad)
        assert ei.value.status == 1
