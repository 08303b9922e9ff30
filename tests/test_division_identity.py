"""The division identity the fp64 row update relies on (rows_mma_block in
paper_2003_03572_b200/csrc/k_rows.inc.cuh): g / h == fma(fma(-g*ri, h, g), ri, g*ri) with
ri = RN(1/h), bit for bit, on 2e7 random pairs (tests/division_identity.c, gcc, C99 fma)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_reciprocal_correction_is_correctly_rounded_division(tmp_path):
    exe = str(tmp_path / "division_identity")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(HERE, "division_identity.c"), "-lm"],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().startswith("0 of ")
