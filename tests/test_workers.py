"""CPU: the multi-device context's worker threads (ws_host.h DevWorkers)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_workers(tmp_path):
    exe = str(tmp_path / "test_workers")
    csrc = os.path.join(ROOT, "paper_2310_17746_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", "-I", csrc,
                    "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_workers.cpp"), "-o", exe,
                    "-L/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout + r.stderr
