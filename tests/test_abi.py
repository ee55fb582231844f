"""The C-ABI library loads and exports every symbol include/emin.h declares
(no compute calls: CPU only), and the package never imports the oracle."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2208_02995_b200.build import build
    build()
    from paper_2208_02995_b200 import load_library
    return load_library()


def header_functions():
    src = open(os.path.join(ROOT, "include", "emin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(emin_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = header_functions()
    for n in ["emin_setup", "emin_iterate", "emin_energy", "emin_get_P"]:
        assert n in names


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (emin_\w+)", out))
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    for n in header_functions():
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(lib):
    lib.emin_status_str.restype = ctypes.c_char_p
    assert lib.emin_status_str(0) == b"EMIN_OK"
    assert lib.emin_status_str(7) == b"EMIN_ERR_BREAKDOWN"


def test_package_does_not_import_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_2208_02995_b200; "
            "assert 'oracle' not in sys.modules; print('ok')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.stdout.strip() == "ok", out.stderr


def test_no_oracle_reference_in_product_sources():
    pkg = os.path.join(ROOT, "paper_2208_02995_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "emin_oracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2208_02995_b200.emin as e\n"
            "e.LIB_PATH = %r\n"
            "try:\n    e.load_library()\nexcept RuntimeError as x:\n    print('raised')\n" %
            (ROOT, str(tmp_path / "nope.so")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert "raised" in out.stdout, out.stderr


def test_opts_and_report_layout_match_header():
    """The ctypes mirrors of emin_opts / emin_report_t have the C sizes."""
    import ctypes as C
    import subprocess
    import tempfile
    from paper_2208_02995_b200 import emin as E
    src = ('#include <stdio.h>\n#include "%s/include/emin.h"\n'
           'int main(){printf("%%zu %%zu", sizeof(emin_opts), sizeof(emin_report_t));}\n' % ROOT)
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "s.c"), "w").write(src)
        subprocess.check_call(["gcc", os.path.join(d, "s.c"), "-o", os.path.join(d, "s")])
        out = subprocess.check_output([os.path.join(d, "s")]).decode().split()
    assert [int(x) for x in out] == [C.sizeof(E.emin_opts), C.sizeof(E.emin_report_t)]
