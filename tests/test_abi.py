"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/annkit_b200.h declares, its host-side helpers reproduce the
reference's bytes, and compute entry points fail loudly without a device
(there is no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1609_07228_b200 as A
from paper_1609_07228_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "annkit_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(annk_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    syms = header_symbols()
    assert len(syms) >= 40
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in annkit_b200.h but not exported"
    assert sorted(syms) == sorted(_lib.EXPORTED), "binding table and header disagree"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_gen_synthetic_matches_reference_bytes():
    from oracle import oracle as O
    o = O.load("oracle")
    assert np.array_equal(A.gen_synthetic(200, 9, 5), o.gen_synthetic(200, 9, 5))


def test_gen_mixture_deterministic_and_shaped():
    a = A.gen_mixture(3000, 16, 10, 0.0, 128.0, 16.0, 0.0, 255.0, True, 1, 1)
    b = A.gen_mixture(3000, 16, 10, 0.0, 128.0, 16.0, 0.0, 255.0, True, 1, 1)
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 255 and np.all(a == np.round(a))
    q = A.gen_mixture(100, 16, 10, 0.0, 128.0, 16.0, 0.0, 255.0, True, 1, 2)
    assert not np.array_equal(q, a[:100])
    f = A.gen_mixture(500, 8, 5, 0.05, 0.35, 0.05, 0.0, 1.0, False, 3, 1)
    assert f.min() >= 0.0 and f.max() <= 1.0


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure mode")
def test_compute_fails_loudly_without_device():
    with pytest.raises(A.AnnkError):
        A.VectorSet(np.zeros((4, 4), np.float32))


def test_host_argument_validation_without_device():
    # validation that happens before any device work still maps to the reference's exception types
    with pytest.raises(A.InvalidArgument):
        A.recall(np.array([1, 2]), np.array([1]))
    with pytest.raises(A.InvalidArgument):
        A.graph_accuracy(np.zeros((2, 3), np.uint32), np.zeros((2, 2), np.uint32))
    assert A.recall(np.array([1, 2, 5, 6]), np.array([1, 2, 3, 4])) == 0.5
