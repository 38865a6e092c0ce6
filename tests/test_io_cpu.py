"""CPU: host formats of the C++ API (OBJ / PNG, cpp/io_b200.cpp) through the
C++ test binary build/test_io_cpu (tests/cpp/test_io_cpu.cpp); the reference's
own test_io.cpp runs against the same code on the GPU box
(tests/test_cpp_api.py)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_formats():
    exe = os.path.join(ROOT, "build", "test_io_cpu")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "test cases passed" in r.stdout
