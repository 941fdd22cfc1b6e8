"""The C-ABI library loads, exports every symbol include/alert_b200.h
declares, and fails loudly (no CPU fallback) without a GPU."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "alert_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(alert_\w+)\(", text, re.M)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "alert_run" in syms and "alert_table_create" in syms and len(syms) >= 18


def test_library_exports_every_declared_symbol():
    from paper_1911_00119_b200 import _lib

    if not _lib.LIB_PATH.exists():
        import __graft_entry__

        __graft_entry__.build()
    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared_symbols())


def test_abi_struct_sizes_match_header():
    from paper_1911_00119_b200 import abi

    assert C.sizeof(abi.AlertSpec) == 64
    assert C.sizeof(abi.AlertFilterConfig) == 80
    assert C.sizeof(abi.AlertPrediction) == 56
    assert C.sizeof(abi.AlertOutputs) == 8 * 7 + 8 + 8 * 4 + 8 * 4
    assert C.sizeof(abi.AlertTrace) == 8 + 8 + 8 * 4 + 8 + 8 * 5 + 8 + 8 * 3
    assert C.sizeof(abi.AlertSpaceDesc) == 8 + 8 * 6 + 8 + 8
    assert C.sizeof(abi.AlertState) == 8 * 10


def test_version_and_strerror():
    from paper_1911_00119_b200 import _lib

    L = _lib.load()
    assert L.alert_abi_version() == 4
    assert L.alert_strerror(-3) == b"invalid constraint spec"


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1911_00119_b200 as A

    with pytest.raises(RuntimeError, match="CUDA"):
        A.get_engine(0)
    from paper_1911_00119_b200 import _lib

    h = C.c_void_p()
    assert _lib.load().alert_create(C.byref(h), 0) == -5  # ALERT_ERR_CUDA
