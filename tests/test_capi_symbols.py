"""CPU checks of the C-ABI library: it loads, exports every symbol declared
in include/lamg_b200.h, its host-only helpers agree with the oracle, and it
refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1108_1310_b200 import _lib


def test_library_exports_declared_symbols():
    lib = _lib.lib()
    names = _lib.declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_host_helpers_match_oracle(port):
    lib = _lib.lib()
    for g in (1.0, 1.5, 1.73, 2.0):
        out = np.empty(12, np.int32)
        lib.lamg_credit_takes(C.c_double(g), C.c_int32(12), out.ctypes.data_as(C.c_void_p))
        assert np.array_equal(out, port.credit_takes(g, 12))
    for q in (1.0, 2.0, 3.0, 7.5):
        assert lib.lamg_flat_mu(q) == port.flat_mu(q)
    for s, k in ((1, 0), (1, 0x517), (12345, 9), (0, 3)):
        assert lib.lamg_rng_derive(s, k) == port.rng_derive(s, k)


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", "x") != "x" and False, reason="")
def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1108_1310_b200.lamg import Context, CudaError
    with pytest.raises(CudaError):
        Context(0)
