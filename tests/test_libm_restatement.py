"""CPU suite: host-compiled checks of restated arithmetic. csrc/glibc_libm.h -- the latent scorer's log and cos, restating
glibc 2.39's x86-64 FMA builds (the reference's std::log / std::cos on these
hosts, rng.cpp:30-36) -- compiled for the host and compared bit for bit with
the host libm on 2^22 draws of the reference's own argument distributions plus
wide random arguments and branch edges (tests/libm_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2411_15381_b200", "csrc")


def _glibc_matches():
    p = "/lib/x86_64-linux-gnu/libm.so.6"
    if not os.path.exists(p):
        return False
    r = subprocess.run(["python3", os.path.join(ROOT, "tools", "extract_libm_fma.py"), p,
                        "--check"], capture_output=True, text=True)
    return r.returncode == 0


@pytest.mark.skipif(not _glibc_matches(), reason="host libm is not the restated glibc build")
def test_log_cos_bit_identical_to_host_libm(tmp_path):
    exe = tmp_path / "libm_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "libm_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), str(1 << 22)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "log: 0 /" in r.stdout and "cos: 0 /" in r.stdout


def test_mt64_jump_ahead_matches_direct_generation(tmp_path):
    """csrc/gf2_jump.h (K8's jump-ahead over the characteristic polynomial in
    csrc/mt64_charpoly.h): jumped states equal direct std::mt19937_64
    generation (tests/mt_jump_check.cpp)."""
    exe = tmp_path / "mt_jump_check"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "mt_jump_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 state words differ" in r.stdout


def test_mt64_charpoly_rederived(tmp_path):
    """tools/mt64_charpoly.cpp re-derives the committed polynomial
    (Berlekamp-Massey on the engine's output; the recurrence is checked on all
    64 bit positions)."""
    exe = tmp_path / "cp"
    subprocess.run(["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tools", "mt64_charpoly.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    with open(os.path.join(CSRC, "mt64_charpoly.h")) as f:
        assert f.read() == r.stdout
