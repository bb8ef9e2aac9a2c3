"""CPU check (no GPU) of the identity behind K3's DFMA total chain
(curve.cu total_run): tools/dfma_lemma.c restates the run test and checks it
against the two-rounding step with the host libm's fma on random steps and
whole chains."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dfma_step_identity_and_run_test(tmp_path):
    exe = tmp_path / "dfma_lemma"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", os.path.join(ROOT, "tools", "dfma_lemma.c"),
                    "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "300000"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    words = out.stdout.split()
    assert int(words[1]) > 1_000_000 and words[3] == "0" and words[7] == "0", out.stdout
