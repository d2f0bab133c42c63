"""CPU tests of the C ABI: the library loads, exports every symbol that
include/ktb.h declares, and reports errors through ktb_last_error. No
compute call is made (no GPU here)."""
import ctypes as C
import subprocess

import pytest

from paper_2405_01599_b200 import _lib


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_version_and_error_channel():
    L = _lib.load()
    assert L.ktb_version() == 1
    cnt = C.c_int(-1)
    rc = L.ktb_device_count(C.byref(cnt))
    if rc != 0:  # no GPU in this container: a CUDA error, with a message
        assert rc == 2 and L.ktb_last_error()
    else:
        assert cnt.value >= 0


def test_contract_errors_before_any_device_work():
    """csr.hpp:38-54 validation happens on the host arrays, with the
    reference's messages, before the device is touched."""
    import numpy as np

    from paper_2405_01599_b200 import ktune as K

    bad = K.CsrMatrix(2, np.array([0, 2, 2]), np.array([1, 0]), np.ones(2))
    with pytest.raises(K.Error, match="columns not strictly increasing"):
        bad.validate()
    bad = K.CsrMatrix(2, np.array([0, 1, 2]), np.array([0, 7]), np.ones(2))
    with pytest.raises(K.Error, match="column index out of range"):
        bad.validate()
    bad = K.SymCsrMatrix(2, np.array([0, 1, 2]), np.array([0, 0]), np.ones(2))
    with pytest.raises(K.Error, match="entry below the diagonal"):
        bad.validate()
    bad = K.CsrMatrix(2, np.array([0, 1]), np.array([0]), np.ones(1))
    with pytest.raises(K.Error, match="row_ptr length"):
        bad.validate()
    with pytest.raises(K.Error, match="num_workers must be >= 1"):
        K.build_row_partition(bad, 0, K.PartitionScheme.row_based)
