"""The C-ABI library loads on a CPU-only host and exports exactly what
include/ircur_b200.h declares (no compute calls: there is no GPU here)."""

import ctypes as C
import os
import re

import pytest

from paper_2010_07422_b200 import _capi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ircur_b200.h")


def _declarations():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    decls = {}
    for m in re.finditer(r"^(?:int|const char\*)\s+(ircur_\w+)\s*\(([^;]*?)\)\s*;", src, flags=re.M | re.S):
        args = m.group(2).strip()
        n = 0 if args in ("", "void") else args.count(",") + 1
        decls[m.group(1)] = n
    return decls


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_capi.LIB_PATH):
        from paper_2010_07422_b200 import _build
        _build.build()
    return _capi.load()


def test_header_and_binding_agree():
    decls = _declarations()
    assert len(decls) >= 20
    protos = {name: len(args) for name, _, args in _capi.PROTOTYPES}
    assert decls == protos


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(_capi.LIB_PATH)
    for name in _declarations():
        assert hasattr(raw, name), name


def test_host_only_entry_points(lib):
    assert lib.ircur_abi_version() == 1
    h = C.c_void_p()
    # argument validation happens before any CUDA call
    rc = lib.ircur_ctx_create(C.byref(h), 0, 7, 10, 10, 2, 5, 5, 10, 0, 10, None)
    assert rc == _capi.EINVAL and h.value is None
    assert b"dtype" in lib.ircur_last_error()
    rc = lib.ircur_ctx_create(C.byref(h), 0, _capi.F64, 0, 10, 2, 5, 5, 10, 0, 10, None)
    assert rc == _capi.EEMPTY
    with pytest.raises(ValueError):
        _capi.check(rc)
    assert lib.ircur_ctx_destroy(None) == _capi.OK
    assert lib.ircur_poll(None, None, None) == _capi.EINVAL


def test_no_fallback_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_capi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_capi, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _capi.load()
