"""CPU-only checks of the C-ABI boundary: the library builds, loads without a
GPU, and exports every symbol include/dcp_capi.h declares."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"DCP_API\s+[\w\s\*]+?\b(dcp_\w+)\s*\(", h.read_text()))
    return names


def test_header_declares_entry_points():
    assert "dcp_splitkv_decode_attn" in _declared()


def test_library_exports_every_declared_symbol():
    from paper_2605_21100_b200 import _capi
    L = _capi.lib()
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    # and the ctypes signature table covers them all
    assert _declared() <= set(_capi.exported_symbols())


def test_no_gpu_is_a_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_21100_b200.attention import DcpContext
    with pytest.raises(Exception):
        DcpContext(0)
