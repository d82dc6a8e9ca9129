"""The C-ABI library loads and exports every entry point include/*.h declares
(no compute calls: this runs on the CPU-only build box)."""
import ctypes
import glob
import os
import re

import pytest

from ccb_helpers import ROOT

LIB = os.path.join(ROOT, "paper_2502_15734_b200", "_lib", "libcc_b200.so")


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names.update(re.findall(r"^CC_API\s+[\w\s\*]+?\b(cc_\w+)\s*\(", src, flags=re.M))
    return sorted(names)


def test_header_declares_the_path():
    names = declared_symbols()
    for must in ("cc_gather_rope_kv", "cc_gemm", "cc_gemm_qkv_rope", "cc_attention", "cc_segment_mass", "cc_chunk_stats",
                 "cc_topk_select", "cc_logits_argmax", "cc_extract_to_pool", "cc_rope_apply_f64"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="native library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.cc_abi_version.restype = ctypes.c_int
    assert lib.cc_abi_version() == 1


def test_binding_table_matches_header():
    from paper_2502_15734_b200 import _native

    assert set(_native._SIGS) == set(declared_symbols())
