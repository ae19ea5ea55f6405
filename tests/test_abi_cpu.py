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
    assert L.pdg_abi_version() == 3


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


def test_invalid_arguments_rejected_before_any_device_work():
    """Argument validation happens on the host, before any CUDA call: every
    entry point returns PDG_EINVAL (1) with a message, no exception crosses
    the ABI."""
    import ctypes as C

    from paper_2506_14851_b200 import _build, _lib
    _build.build()
    L = _lib.load()
    EINVAL = 1
    null = None
    assert L.pdg_gittins_rank_f64(null, null, null, -1, 4, null, null) == EINVAL
    assert L.pdg_gittins_rank_f64_host(null, null, null, 3, 0, null, null) == EINVAL
    assert L.pdg_policy_keys(7, null, null, null, null, null, C.c_double(0.0), 10, null, null,
                             null, null) == EINVAL
    assert L.pdg_policy_keys(2, null, null, null, null, null, C.c_double(0.0), 10, null, null,
                             null, null) == EINVAL
    assert L.pdg_dispatch_plan(null, null, null, null, null, null, -1, null, 1,
                               C.c_double(1.5), 1, 3, null, null, null, null, 0, null) == EINVAL
    assert L.pdg_order(null, null, null, null, 5, 16, null, 0, null) == EINVAL
    assert L.pdg_order_update(null, null, null, 4, null, 9, null, null, null, null, 0,
                              null) == EINVAL
    assert L.pdg_pearson_flags(null, null, null, null, -2, C.c_double(0.5), null, null,
                               null) == EINVAL
    assert L.pdg_prewarm_window_index(null, 1, null, 4, null, null) == EINVAL
    assert L.pdg_mc_remaining_demand(null, null, 1, 512, 64, 64, 0, 0, null, null, 0,
                                     null) == EINVAL
    msg = L.pdg_last_error()
    assert msg and b"pdg_mc_remaining_demand" in msg
