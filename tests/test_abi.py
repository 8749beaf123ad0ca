"""Host-side checks of the C ABI boundary (no GPU needed): the library loads, exports
every symbol include/rtucker.h declares, and rejects invalid arguments before touching
the device."""
import ctypes as C
import os
import re

import pytest

from paper_1905_07311_b200 import build as B
from paper_1905_07311_b200 import rtucker as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtucker.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return R.load_library()


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rtucker_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("rtucker_hosvd", "rtucker_sthosvd", "rtucker_adaptive", "rtucker_sparse_sthosvd",
              "rtucker_ctx_create", "rtucker_result_free"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert names
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(R.EXPORTED)


def test_exports_are_c_symbols(lib):
    """extern "C": unmangled names, visible via dlsym."""
    out = os.popen(f"nm -D --defined-only {R.LIB_PATH}").read()
    for n in _declared():
        assert re.search(rf"\bT {n}\b", out), n


def test_version(lib):
    assert b"sm_100a" in lib.rtucker_version()


def test_invalid_arguments_without_gpu(lib):
    h = C.c_void_p()
    na, nf = R.ALLOC_FN(), R.FREE_FN()
    assert lib.rtucker_ctx_create(0, None, None, 0, 0, na, nf, None, C.byref(h)) == 1      # nranks < 1
    assert lib.rtucker_ctx_create(0, None, None, 2, 2, na, nf, None, C.byref(h)) == 1      # rank >= nranks
    assert lib.rtucker_ctx_create(0, None, None, 0, 2, na, nf, None, C.byref(h)) == 1      # no NCCL id for 2 ranks
    # allocation hooks come in pairs
    a_only = R.ALLOC_FN(lambda n, s, u: None)
    assert lib.rtucker_ctx_create(0, None, None, 0, 1, a_only, nf, None, C.byref(h)) == 1
    out = C.POINTER(R.ResultStruct)()
    desc = R.DenseDesc()
    ranks = (C.c_int64 * 3)(1, 1, 1)
    assert lib.rtucker_sthosvd(None, C.byref(desc), ranks, 0, 0, None, 0, C.byref(out)) == 1
    assert lib.rtucker_hosvd(None, C.byref(desc), ranks, 0, 0, 0, C.byref(out)) == 1
    assert lib.rtucker_adaptive(None, C.byref(desc), 0.1, 1, None, None, 0, 0, C.byref(out)) == 1
    assert lib.rtucker_last_error(None) == b"null context"
    assert lib.rtucker_launch_count(None) == 0


def test_struct_layout_matches_header(lib):
    """ctypes mirrors of the descriptors have the C layout (offsets from a tiny C probe)."""
    import subprocess
    import tempfile
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "rtucker.h"
int main(){
 printf("%zu %zu %zu %zu\n", sizeof(rtucker_dense_desc), offsetof(rtucker_dense_desc,data),
        sizeof(rtucker_coo_desc), offsetof(rtucker_coo_desc,vals));
 printf("%zu %zu %zu %zu %zu\n", sizeof(rtucker_result), offsetof(rtucker_result,core),
        offsetof(rtucker_result,norm_sq), offsetof(rtucker_result,selection), offsetof(rtucker_result,internal));
 return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "probe.c")
        open(p, "w").write(src)
        exe = os.path.join(d, "probe")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), p, "-o", exe])
        a, b = subprocess.check_output([exe]).decode().splitlines()
    a = [int(t) for t in a.split()]
    b = [int(t) for t in b.split()]
    assert a == [C.sizeof(R.DenseDesc), R.DenseDesc.data.offset, C.sizeof(R.CooDesc), R.CooDesc.vals.offset]
    assert b == [C.sizeof(R.ResultStruct), R.ResultStruct.core.offset, R.ResultStruct.norm_sq.offset,
                 R.ResultStruct.selection.offset, R.ResultStruct.internal.offset]


def test_product_path_does_not_import_the_oracle():
    """The product package never references oracle/ (independence)."""
    pkg = os.path.join(ROOT, "paper_1905_07311_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
