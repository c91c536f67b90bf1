"""Builds and runs tests/cpp/host_unit.cpp (C++ cases mirroring the reference's
test_sched.cpp / test_kvcache.cpp / test_core.cpp) against the host sources."""
import glob
import os
import shutil
import subprocess
import tempfile

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_host_unit_cpp():
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2403_02310_b200/csrc/host/*.cpp")))
    srcs = [s for s in srcs if not s.endswith(("capi.cpp", "descriptor.cpp"))]
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "host_unit")
        subprocess.run([cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "paper_2403_02310_b200/csrc/host"),
                        os.path.join(ROOT, "tests/cpp/host_unit.cpp"), *srcs, "-o", exe], check=True)
        r = subprocess.run([exe], capture_output=True, text=True)
        print(r.stdout)
        assert r.returncode == 0, r.stdout
