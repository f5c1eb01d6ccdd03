"""Host expander of the 8-bit enumeration wire format (csrc/ws_wire.cpp) on
CPU: random block layouts, output alignments and partial ranges, AVX-512 and
AVX-512 without IFMA and scalar paths (the GPU side is covered by the enumeration parity tests, which
take the wire path for every multi-chunk host enumeration)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2310_17746_b200", "csrc")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("wire") / "test_wire")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-pthread", "-I", CSRC,
                    os.path.join(ROOT, "tests", "cpp", "test_wire.cpp"),
                    os.path.join(CSRC, "ws_wire.cpp"), "-o", out], check=True)
    return out


@pytest.mark.parametrize("isa", ["ifma", "avx512", "scalar"])
def test_wire_expand(exe, isa):
    env = dict(os.environ, WHEELSIEVE_HOST_SCALAR=str(int(isa == "scalar")),
               WHEELSIEVE_HOST_NO_IFMA=str(int(isa == "avx512")))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
