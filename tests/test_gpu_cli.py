"""GPU: the CLI mirror (tools/wheelsieve_gpu.py), cases from the reference's
test_cli.cpp (cited per test)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = [sys.executable, os.path.join(ROOT, "tools", "wheelsieve_gpu.py")]


def run(*args):
    r = subprocess.run(CLI + list(args), capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout


def test_summary_line():  # test_cli.cpp:68-85
    rc, out = run("sieve", "--limit", "30", "--count-only")
    assert rc == 0 and out.startswith("count=10 largest=29 ms=")
    rc, out = run("sieve", "--limit", "30")
    assert rc == 0 and out.splitlines()[:10] == ["2", "3", "5", "7", "11", "13", "17", "19", "23", "29"]


@pytest.mark.parametrize("limit", [30, 10_000, 1_000_000])
def test_verify_pass(limit):  # test_cli.cpp:87-103
    rc, out = run("verify", "--limit", str(limit))
    assert rc == 0 and out.startswith("PASS")


def test_verify_poison():  # test_cli.cpp:117-121
    rc, out = run("verify", "--limit", "10000", "--poison")
    assert rc == 1 and "FAIL first divergence at index 24: expected 97, got 101" in out


def test_usage_exit_code():  # test_cli.cpp:123-141
    rc, _ = run("sieve")
    assert rc == 2


def test_store_and_bench(tmp_path):  # test_cli.cpp:143-227
    d = str(tmp_path / "s")
    rc, out = run("sieve", "--limit", "100000", "--out", d, "--format", "binary",
                  "--primes-per-file", "1000")
    assert rc == 0 and out.startswith("count=9592 largest=99991")
    assert os.path.exists(os.path.join(d, "manifest.json"))
    csv = str(tmp_path / "b.csv")
    rc, _ = run("bench", "--limits", "1000", "100000000", "--segment-slots", "4096", "262144",
                "--repeats", "2", "--csv", csv)
    lines = open(csv).read().splitlines()
    assert rc == 0
    assert lines[0] == "threads,limit,segment_span,flag_width,wall_ms,iterations,peak_flag_bytes,prime_count"
    assert len(lines) == 5 and lines[-1].endswith(",5761455")
