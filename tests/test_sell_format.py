"""CPU tests of the resident device formats: the SELL-16 / packed SELL-P host
encoders in paper_1612_09447_b200/csrc/host_sell.cpp round-trip every CSR entry
through the kernels' index arithmetic (tests/cpp/test_sell.cpp), and the
blocked K(x)x scatter structure (tests/cpp/test_kxblock.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sell_encoders_round_trip(tmp_path):
    exe = tmp_path / "test_sell"
    csrc = os.path.join(ROOT, "paper_1612_09447_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", "-fopenmp", "-I" + csrc, "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_sell.cpp"), os.path.join(csrc, "host_sell.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


def test_kx_blocks_emulated_scatter(tmp_path):
    exe = tmp_path / "test_kxblock"
    csrc = os.path.join(ROOT, "paper_1612_09447_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", "-fopenmp", "-I" + csrc, os.path.join(ROOT, "tests", "cpp",
                    "test_kxblock.cpp"), os.path.join(csrc, "host_kxblock.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
