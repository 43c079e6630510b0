"""Host unit test of the product's exact clock aggregation and memory-profile
composition (csrc/exact_add.cuh): bit-identical to plain IEEE adds (random,
tie-heavy dyadic and zero costs; binade crossings; chunked repetitions)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_exact_add_matches_plain_adds(tmp_path):
    exe = str(tmp_path / "exact_add_check")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off",
                           "-o", exe, os.path.join(HERE, "native", "exact_add_check.cpp")])
    out = subprocess.run([exe, "1500"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout
