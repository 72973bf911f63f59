"""The C-ABI library loads on CPU and exports every symbol include/attn_b200.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

from conftest import ROOT
from paper_2502_15349_b200 import build, runtime

HEADER = ROOT / "include" / "attn_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(af_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("af_parallel_fwd", "af_parallel_bwd", "af_parallel_bwd_workspace",
                     "af_linear_fwd", "af_linear_bwd", "af_mla_decode", "af_status_string",
                     "af_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib_path = build.build_library()
    handle = ctypes.CDLL(str(lib_path))
    for name in declared_functions():
        assert hasattr(handle, name), name


def test_runtime_binds_every_declared_symbol():
    assert sorted(runtime.SIGNATURES) == declared_functions()
    lib = runtime.lib()
    assert lib.af_status_string(runtime.AF_ERR_UNSUPPORTED) == b"unsupported"
    assert lib.af_status_string(runtime.AF_ERR_NAN) == b"nan-in-output"


def test_descriptor_validation_without_gpu():
    # input errors are raised before any device work, so they are checkable on CPU
    lib = runtime.lib()
    d = runtime.ParallelDesc()
    d.batch = 1; d.heads_q = 3; d.heads_kv = 2; d.seq_q = d.seq_k = 8; d.d_qk = d.d_v = 64
    st = lib.af_parallel_fwd(d, None, None, None, None, None, None)
    assert st == runtime.AF_ERR_SHAPE
    assert b"multiple" in lib.af_last_error()
    with pytest.raises(Exception):
        runtime.check(st, "af_parallel_fwd")
