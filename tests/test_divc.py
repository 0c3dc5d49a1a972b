"""The update kernels divide by the bias corrections (Alg. 5 l.14-15,
PAPER.md:287-288) with Markstein's two-FMA correction of a reciprocal product
(device.cuh divc, R21) instead of the IEEE division sequence.  This
CPU test emulates that arithmetic in C (fmaf, no contraction) and checks it
against the IEEE quotient a / b bit for bit for the divisors every step uses,
b = fl32(1 - beta^t), beta in {0.9, 0.999}, t up to 2e5, and random a over
2^-100 .. 2^60 (the kernel sends smaller |a| to the IEEE division)."""
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))


def test_divc_matches_ieee_division():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "divc_check")
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-o", exe,
                               os.path.join(HERE, "native", "divc_check.c"), "-lm"])
        r = subprocess.run([exe, "2000"], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "bad 0" in r.stdout
