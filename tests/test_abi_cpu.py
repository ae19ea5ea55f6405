"""CPU-side checks of the C-ABI library: it loads, exports every declared
symbol, and the product refuses to run without a CUDA device."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "pdg_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(pdg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_2506_14851_b200 import _build, _lib
    _build.build()
    L = _lib.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert set(declared_symbols()) == set(_lib.EXPORTS)
    assert L.pdg_abi_version() == 2


def test_sm100a_cubin_in_library():
    import subprocess
    from paper_2506_14851_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="GPU present")
def test_no_cpu_fallback():
    import numpy as np
    from paper_2506_14851_b200 import sched
    from paper_2506_14851_b200._lib import PdgDeviceError
    with pytest.raises(PdgDeviceError):
        sched.gittins_rank_batch(np.ones((1, 2)), np.full((1, 2), 0.5), np.zeros(1))
