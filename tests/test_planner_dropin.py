"""The reference's own acceptance suite, compiled UNCHANGED against the
product's drop-in header.

/root/reference/proj/tests/acceptance.cpp (criteria 1-8 of the reference
SPEC) includes "reforward/reforward.hpp"; tests/dropin/reforward/*.hpp are
one-line shims that serve every reference header name from
include/reforward_b200/planner.hpp.  The binary links libreforward_b200.so
(the product planner) and must print "ACCEPTANCE: 8/8".  Runs only where the
reference tree exists (this container); the source is read in place, never
copied.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
LIB_DIR = os.path.join(ROOT, "paper_1808_00079_b200")


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_TESTS, "acceptance.cpp")),
                    reason="reference tree not present")
def test_reference_acceptance_suite_against_dropin_header(tmp_path):
    exe = tmp_path / "acceptance"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'tests', 'dropin')}", f"-I{REF_TESTS}",
           f"-I{os.path.join(ROOT, 'include')}", os.path.join(REF_TESTS, "acceptance.cpp"), "-o", str(exe),
           f"-L{LIB_DIR}", "-lreforward_b200", f"-Wl,-rpath,{LIB_DIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert "ACCEPTANCE: 8/8 criteria passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0
