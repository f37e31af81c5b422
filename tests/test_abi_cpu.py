"""CPU-side checks of the C-ABI boundary (no GPU compute): the library loads, exports every
symbol include/cssar.h declares, maps error codes, and the product package does not touch
oracle/."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cssar.h")
PKG = os.path.join(ROOT, "paper_1302_3120_b200")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cssar_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("cssar_plan_create", "cssar_forward", "cssar_adjoint", "cssar_ita_iterate", "cssar_image"):
        assert name in d


def test_library_exports_every_declared_symbol():
    from paper_1302_3120_b200 import cssar
    lib = cssar.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(cssar.SYMBOLS)


def test_error_strings_without_gpu():
    from paper_1302_3120_b200 import cssar
    lib = cssar.load_library()
    assert lib.cssar_error_string(0) == b"ok"
    assert b"k" in lib.cssar_error_string(-3)
    for code in cssar.ERRORS:
        assert lib.cssar_error_string(code) != b"unknown error"


def test_null_plan_is_rejected_without_gpu():
    from paper_1302_3120_b200 import cssar
    lib = cssar.load_library()
    assert lib.cssar_plan_destroy(None) == -10
    n = ctypes.c_size_t()
    assert lib.cssar_workspace_size(None, ctypes.byref(n)) == -10
    assert lib.cssar_plan_set_pulse(None, None, 0) == -10
    it = ctypes.c_int32()
    assert lib.cssar_ita_iters_done(None, ctypes.byref(it)) == -10


def test_product_path_does_not_use_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "oracle." not in src.replace("oracle/", ""), f


def test_sm100a_code_in_library():
    """The shipped library carries sm_100a SASS (cuobjdump), not a PTX-only JIT image."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    lib = os.path.join(PKG, "libcssar.so")
    out = subprocess.run([cuobjdump, "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_params_validation_without_gpu():
    """cssar_plan_create validates before any CUDA call: operator code and the RDA window
    bound (include/cssar.h cssar_op: (1/D_max - 1) n_rg < 1/2)."""
    from inputs.configs import SarParams
    from paper_1302_3120_b200 import cssar
    lib = cssar.load_library()
    h = ctypes.c_void_p()
    bad_op = cssar._params_c(SarParams(n_az=256, n_rg=256))
    bad_op.op = 7
    assert lib.cssar_plan_create(ctypes.byref(h), ctypes.byref(bad_op), 1, 0, None, None) == -1
    # prf 4000 Hz at 16384 gates: the RDA migration varies by 0.53 cell across the row
    wide = cssar._params_c(SarParams(n_az=256, n_rg=16384, Fr=120e6, prf=4000.0), "rda")
    assert lib.cssar_plan_create(ctypes.byref(h), ctypes.byref(wide), 1, 0, None, None) == -1
    assert not h.value


def test_log_csv_export(tmp_path):
    import csv
    from paper_1302_3120_b200.cssar import write_log_csv
    entries = [dict(sigma=1.5, lam=1.5, mu=1.0, support=5, resid2=2.25), dict(sigma=0.5, lam=0.5, mu=1.0, support=4,
                                                                                 resid2=1.0)]
    path = tmp_path / "log.csv"
    write_log_csv(entries, path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["iter", "sigma", "lambda", "mu", "support", "resid2"]
    assert [float(r[1]) for r in rows[1:]] == [1.5, 0.5] and rows[2][4] == "4"
