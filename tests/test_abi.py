"""CPU-side checks of the C ABI boundary (no GPU needed): the library loads,
exports every entry point include/skv_b200.h declares, carries sm_100a code,
does not link the oracle, and its host-side rules (k, m, argument checks)
match the oracle / reference."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skv_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2403_17312_b200._lib import lib as load

    return load()


def declared():
    src = "\n".join(ln for ln in open(HEADER).read().splitlines() if not ln.lstrip().startswith("typedef"))
    return sorted(set(re.findall(r"\b(skv_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name


def test_library_is_sm100a_and_oracle_free():
    from paper_2403_17312_b200._lib import SO_PATH

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", SO_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    syms = subprocess.run(["nm", "-D", SO_PATH], capture_output=True, text=True).stdout
    assert " oc_" not in syms and " ref_" not in syms


def test_window_k_matches_oracle(lib, port, golden):
    for n in golden["k_n"]:
        for r in golden["k_r"]:
            assert lib.skv_swa_window_k(int(n), float(r)) == port.swa_window_k(int(n), float(r))
            assert lib.skv_swa_keep_count(int(n), float(r)) == port.swa_keep_count(int(n), float(r))
    assert lib.skv_swa_window_k(10, 0.0) == 0
    assert b"ratio out of (0,1]" in lib.skv_last_error()


def test_argument_errors_map_to_reference_classes(lib):
    from paper_2403_17312_b200._lib import ContractViolation, Unsupported, check
    from paper_2403_17312_b200.api import _Desc

    with pytest.raises(ContractViolation):
        check(lib.skv_cache_create(None, None))
    d = _Desc(1, 1, 4, 64, 8, 1, 1, 0, 0)
    h = C.c_void_p()
    with pytest.raises(Unsupported):
        check(lib.skv_cache_create(C.byref(d), C.byref(h)))
    d = _Desc(1, 1, 4, 128, 8, 3, 3, 0, 0)  # u8 queries are not a compute dtype
    with pytest.raises(Unsupported):
        check(lib.skv_cache_create(C.byref(d), C.byref(h)))
    with pytest.raises(ContractViolation):
        check(lib.skv_top_k_indices(None, 1, 4, 4, 5, None, None))  # k exceeds length
    with pytest.raises(ContractViolation):
        check(lib.skv_quantize(None, 6, 3, 0, None, None, None, None))  # bits


def test_header_is_plain_c(tmp_path):
    """include/skv_b200.h is the FFI boundary for any host language: it must
    compile as strict C99 (no C++ in the signatures) and a C program must
    link against the library's exports."""
    src = tmp_path / "use.c"
    src.write_text('#include "skv_b200.h"\n'
                   "int main(void) {\n"
                   "    skv_cache_desc d = {1, 1, 8, 128, 64, SKV_F16, SKV_F16, 0, 0};\n"
                   "    (void)d;\n"
                   "    return skv_swa_window_k(512, 0.2) == 51 ? 0 : 1;\n"
                   "}\n")
    exe = tmp_path / "use"
    lib_dir = os.path.join(ROOT, "paper_2403_17312_b200")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe), "-L", lib_dir, "-lskv_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    assert subprocess.run([str(exe)]).returncode == 0  # swa_window_k is host code: no GPU needed
