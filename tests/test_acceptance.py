"""The reference's own acceptance program, UNCHANGED, against the GPU library.

tests/cpp/Makefile compiles /root/reference/proj/tests/acceptance.cpp (only
present in the build container) against the drop-in headers
include/wheelsieve/*.hpp and links it to libwheelsieve.so -- no reference code
is linked -- into tests/cpp/_ref/acceptance_gpu (git-ignored, shipped to the
GPU box).  Its CLI criteria drive the drop-in CLI paper_2310_17746_b200/wheelsieve.

Criterion 6 ("scaling") times wall(threads = 1..4) of the reference's CPU
worker pool; on the GPU `threads` only shapes the worker tiles, so that
criterion measures nothing here and is reported, not required."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_ref", "acceptance_gpu")
CLI = os.path.join(ROOT, "paper_2310_17746_b200", "wheelsieve")
REF_SRC = "/root/reference/proj/tests/acceptance.cpp"


def test_acceptance_builds_against_dropin_headers():
    if not os.path.exists(REF_SRC):
        pytest.skip("reference sources absent (GPU box): the binary was built in the container")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "acceptance"],
                   check=True)
    assert os.path.exists(EXE)
    # only our libraries are linked
    libs = subprocess.run(["ldd", EXE], capture_output=True, text=True).stdout
    assert "libwheelsieve.so" in libs and "libwheelsieve_cuda.so" in libs


@pytest.mark.gpu
def test_reference_acceptance_criteria():
    if not os.path.exists(EXE):
        pytest.skip("acceptance_gpu not built (build() compiles it where /root/reference exists)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=1200,
                       cwd=os.path.join(ROOT, "tests", "cpp"))
    lines = r.stdout.splitlines()
    status = {}
    for ln in lines:
        m = re.match(r"\[(PASS|FAIL|SKIP)\] (\d+)\.", ln)
        if m:
            status[int(m.group(2))] = m.group(1)
    print(r.stdout)
    for crit in (1, 2, 3, 4, 5, 7, 8, 9):
        assert status.get(crit) == "PASS", (crit, r.stdout, r.stderr)
    assert status.get(6) in ("PASS", "FAIL", "SKIP")
