"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
the ctypes record layouts match the C structs. No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT


def header_functions(path):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsqfit_cuda_\w+)\s*\(", text)))


def test_capi_exports_every_declared_symbol():
    from paper_1512_08017_b200 import _capi
    lib = _capi.lib()
    declared = header_functions(os.path.join(ROOT, "include", "lsqfit_cuda.h"))
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_capi.exported_symbols()) == declared


def test_library_is_sm100a_only():
    from paper_1512_08017_b200 import _capi
    _capi.lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_kernels_use_bulk_copy_engine():
    """The hot kernel streams HBM->SMEM with cp.async.bulk (SASS UBLKCP)."""
    from paper_1512_08017_b200 import _capi
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun",
                           "_ZN3lsq17power_sums_kernelILi3EEEvNS_6PsArgsE", _capi.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass
    assert "SYNCS" in sass  # mbarrier ops


def test_record_layouts_match_c(tmp_path):
    from paper_1512_08017_b200 import _capi
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "lsqfit_cuda.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(lsqfit_result), '
                   'offsetof(lsqfit_result, n), offsetof(lsqfit_result, status), sizeof(lsqfit_diag), '
                   'offsetof(lsqfit_diag, status));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert got == [_capi.RESULT_BYTES, _capi.Result.n.offset, _capi.Result.status.offset, _capi.DIAG_BYTES,
                   _capi.Diag.status.offset]


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1512_08017_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "liboracle" not in text, f
                assert "lsqfit_oracle.h" not in text and "orc_" not in text, f


@pytest.mark.parametrize("mod", ["paper_1512_08017_b200.lsqfit", "paper_1512_08017_b200.device"])
def test_modules_import_without_gpu(mod):
    __import__(mod)


def test_stated_sum_bound_levels():
    """The power-sum accuracy bound the library states (host-only query)."""
    from paper_1512_08017_b200 import _capi
    # m <= 2: the reference's terms, P = 16 trees + 1 pair add; m >= 3: exact
    # products (8-term DFMA chains, then a tree over 2: 9 levels), + 1 pair
    # add for m = 3, 4; from m = 5 8 tiles per fold (+7), from m = 6 the
    # lane-pair exchange (+1)
    assert [_capi.sum_error_levels(m) for m in range(13)] == [5] * 3 + [10] * 2 + [16] + [17] * 7
    assert [_capi.sum_terms(m) for m in range(13)] == [_capi.TERMS_REFERENCE] * 3 + [_capi.TERMS_PRODUCTS] * 10
    assert _capi.sum_error_levels(-1) == -1 and _capi.sum_error_levels(13) == -1
    assert _capi.sum_terms(-1) == -1 and _capi.sum_terms(13) == -1


def test_argument_validation_without_a_device():
    """Argument checks run on the host before any CUDA call: NULL or invalid
    arguments give LSQFIT_EINVAL (no exception crosses the ABI), and creating
    a context without a GPU reports a CUDA error instead of crashing."""
    import ctypes as C
    from paper_1512_08017_b200 import _capi
    L = _capi.lib()
    EINVAL = _capi.EINVAL
    null = None
    buf = (C.c_double * 4)()
    res = _capi.Result()
    assert L.lsqfit_cuda_fit_host(null, buf, 2, 3, 1, C.byref(res)) == EINVAL
    assert L.lsqfit_cuda_fit_device(null, null, 0, 3, 1, null, null) == EINVAL
    assert L.lsqfit_cuda_power_sums_host(null, buf, 2, 20, buf, buf) == EINVAL
    assert L.lsqfit_cuda_solve_host(null, buf, buf, 2, buf) == EINVAL
    assert L.lsqfit_cuda_solve_sums_host(null, buf, buf, 1, buf) == EINVAL
    assert L.lsqfit_cuda_group_create(null, null, 0) == EINVAL
    assert L.lsqfit_cuda_sum_error_levels(-1) == -1
    assert L.lsqfit_cuda_strerror(EINVAL) == b"invalid argument"
    h = C.c_void_p()
    st = L.lsqfit_cuda_create(C.byref(h), 0)
    if st == _capi.OK:  # a GPU is visible after all
        L.lsqfit_cuda_destroy(h)
    else:
        assert st in (_capi.ECUDA, _capi.ENOMEM) and not h.value
