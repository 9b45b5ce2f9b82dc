"""The C-ABI library loads and exports every symbol include/enova.h declares;
host-side validation works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "enova.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(enova_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2407_09486_b200 import build as B
    B.build()
    from paper_2407_09486_b200 import _lib
    return _lib.lib()


def test_every_declared_symbol_is_exported(L):
    from paper_2407_09486_b200 import _lib
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTS)


def test_shared_object_targets_sm100a_tensor_cores():
    import shutil
    import subprocess
    from paper_2407_09486_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run([tool, "-lelf", _lib.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass             # tcgen05.ld
    assert "UBLKCP" in sass           # bulk async copy


def test_status_strings_and_version(L):
    assert L.enova_abi_version() == 1
    assert L.enova_status_string(0) == b"ENOVA_OK"
    assert L.enova_status_string(4) == b"ENOVA_ERR_TOO_FEW_EXCEEDANCES"


def test_workspace_sizing_and_envelope(L):
    from paper_2407_09486_b200._lib import Detector
    ok = Detector(64, 16, 128, 16)
    assert L.enova_detector_workspace_bytes(C.byref(ok)) >= 128 * 1024 * 2
    for bad in (Detector(63, 16, 128, 16), Detector(64, 12, 128, 16), Detector(64, 16, 96, 16),
                Detector(64, 16, 128, 17), Detector(64, 24, 128, 16)):
        assert L.enova_detector_workspace_bytes(C.byref(bad)) == 0
    a = L.enova_threshold_workspace_bytes(10**8, 0.98)
    b = L.enova_threshold_workspace_bytes(10**6, 0.98)
    assert a > b > 0
    assert a >= 8 * int(0.02 * 10**8)            # the fp64 tail the fit runs on
    assert a >= 4 * 10**8                        # n >= 2^22: sampled selection's candidate segments
    for n in (10**6, 10**8):
        for w in (1, 2, 8):                          # fp64 tail + this rank's fp32 tail + w gathered slots
            c = L.enova_threshold_comm_workspace_bytes(n, 0.98, w)
            assert c >= 8 * int(0.02 * n) + 4 * int(0.02 * n) * (w + 1)
    # the communicator path runs the full radix passes (no candidate buffer)
    assert L.enova_threshold_comm_workspace_bytes(10**6, 0.98, 1) >= b


def test_validation_before_any_launch(L):
    from paper_2407_09486_b200._lib import Detector, Series, Threshold
    det = Detector(64, 16, 128, 16)
    s = Series()
    assert L.enova_score_windows(C.byref(s), C.byref(det), None, 0, None, None, None) == 1
    bad = Detector(63, 16, 128, 16)
    assert L.enova_score_windows(C.byref(s), C.byref(bad), None, 0, None, None, None) == 2
    assert L.enova_prepare_detector(C.byref(det), None, 0, None) == 1       # NULL weights
    thr = Threshold()
    assert L.enova_fit_threshold(None, 10, 10, 0.98, 1e-3, None, C.byref(thr), None, 0, None) == 1
    assert L.enova_fit_threshold(None, 0, 0, 1.5, 1e-3, None, C.byref(thr), None, 0, None) == 1
    assert L.enova_ring_push(None, 1, 64, 16, None, 0, None) == 1
    assert b"NULL" in L.enova_last_error() or len(L.enova_last_error()) > 0
