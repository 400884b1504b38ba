"""CPU checks of the drop-in boundary: the native library loads without a GPU and exports
every entry point declared in include/ttutv_b200.h."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ttutv_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ttg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for required in ["ttg_decompose", "ttg_qr_col_pivot", "ttg_utv", "ttg_svd", "ttg_truncate",
                     "ttg_reconstruct", "ttg_verify_bound", "ttg_result_report"]:
        assert required in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_07904_b200._native import LIB_PATH, SIGNATURES, lib
    assert LIB_PATH.exists(), "run __graft_entry__.build() first"
    handle = lib()
    for name in declared_symbols():
        assert hasattr(handle, name), name
        assert name in SIGNATURES, f"{name} missing from the ctypes signature table"


def test_no_device_reports_zero_or_more():
    from paper_2501_07904_b200._native import lib
    assert lib().ttg_device_count() >= 0
    assert lib().ttg_abi_version() == 1
