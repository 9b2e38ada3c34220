"""The C-ABI library loads here (no GPU needed) and exports exactly what
include/dp_b200.h declares — no compute calls."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dp_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for want in ("dp_copy_strided", "dp_accumulate_strided", "dp_conv_fwd", "dp_conv_dgrad",
                 "dp_conv_wgrad", "dp_attn_fwd_update", "dp_attn_finalize",
                 "dp_attn_bwd_preprocess", "dp_attn_bwd_update", "dp_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2605_11111_b200 import _lib

    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers the same set
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_library_is_sm100a_only():
    from paper_2605_11111_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_abi_version_without_gpu():
    from paper_2605_11111_b200 import _lib

    lib = _lib.load()
    assert lib.dp_abi_version() == 1
