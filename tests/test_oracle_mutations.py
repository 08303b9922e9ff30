"""Mutation check of the oracle's pins (CPU): each case compiles a copy of
oracle/sacd_oracle.c with ONE plausible mistake (a dropped term, a wrong sign or index, a
transposed operand, a reversed gate) and runs tests/test_oracle_pins.py against it in a
subprocess.  The pins must fail for every mutation; a surviving mutation means the part
of the oracle it touches is not pinned.  Test infrastructure only (ORACLE_SRC / ORACLE_LIB
point the oracle wrapper at the mutated copy)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sacd_oracle.c")

# (name, cited passage, original text, replacement, which occurrence (0-based))
MUTATIONS = [
    ("L_frob_replaced_by_h", "Alg 1 L=||H|| (P:568), Eq 20",
     "const double L = (l_mode == 0) ? h : Lfrob;", "const double L = h;", 0),
    ("E_changed_counts_every_selection", "C14 / Lemma 4 (P:830)",
     "if (uhat != 0.0) Ech += 1;", "Ech += 1;", 0),
    ("gradient_sign_of_m", "Eq 14 (P:352), C3",
     "const double g = -m[r] + s;", "const double g = m[r] + s;", 0),
    ("importance_drops_quadratic", "Eq 20 (P:451)",
     "z = -g * uhat - (L / 2.0) * uhat * uhat;", "z = -g * uhat;", 0),
    ("importance_half_L_dropped", "Eq 20 (P:451)",
     "z = -g * uhat - (L / 2.0) * uhat * uhat;", "z = -g * uhat - L * uhat * uhat;", 0),
    ("step_sign", "Eq 11-13 (P:364-376)",
     "fmax(0.0, u[r] - g / h)", "fmax(0.0, u[r] + g / h)", 0),
    ("step_unprojected", "Eq 12-13 projection (P:369-376)",
     "fmax(0.0, u[r] - g / h)", "(u[r] - g / h)", 0),
    ("gate_first_nonstrict", "Alg 1 z>0 (P:576), C7",
     "if (branch == BR_FIRST) sel = z > 0.0;", "if (branch == BR_FIRST) sel = z >= 0.0;", 0),
    ("gate_eq24_reversed", "Eq 24 (P:487)",
     "else if (branch == BR_EQ24) sel = (z - zp[r]) > 0.0;", "else if (branch == BR_EQ24) sel = (zp[r] - z) > 0.0;", 0),
    ("gate_eq27_reversed", "Eq 27 (P:502)",
     "else sel = (zp[r] - z) > 0.0;", "else sel = (z - zp[r]) > 0.0;", 0),
    ("zprev_only_when_selected", "P:598, C8",
     "      zp[r] = z;\n      if (decisions) decisions[i * R + r] = (uint8_t)sel;\n    }\n    free(u0);",
     "      if (sel) zp[r] = z;\n      if (decisions) decisions[i * R + r] = (uint8_t)sel;\n    }\n    free(u0);", 0),
    ("gauss_seidel_replaced_by_jacobi", "C9",
     "for (int j = 0; j < R; j++) s += (jacobi ? u0[j] : u[j]) * H[j * R + r];",
     "for (int j = 0; j < R; j++) s += ((r > 0 && j < r) ? u[j] * 0.999 : u[j]) * H[j * R + r];", 0),
    ("ti_sums_factors", "Eq 25 (P:493)",
     "for (int64_t x = 0; x < I * R; x++) ti += zprev[x];", "for (int64_t x = 0; x < I * R; x++) ti += F[x];", 0),
    ("branch_rule_reversed", "Eq 26-27 (P:495-502), C10",
     "(ti_hist[k - 2] > ti_hist[k - 3]) ? BR_EQ27 : BR_EQ24", "(ti_hist[k - 2] > ti_hist[k - 3]) ? BR_EQ24 : BR_EQ27", 0),
    ("mttkrp_b_indexed_by_a", "Eq 9 (P:340), P:623-625",
     "B[(int64_t)idx_b[e] * R + r]", "B[(int64_t)idx_a[e] * R + r]", 0),
    ("mttkrp_value_dropped", "Eq 9 (P:340)",
     "((double)val[e] * A[", "((double)1.0 * A[", 0),
    ("hadamard_drops_factor", "Eq 10 (P:345)",
     "Z[i] = X[i] * Y[i];", "Z[i] = X[i];", 0),
    ("gram_uses_one_column", "Eq 10 (P:345)",
     "s += F[i * R + r] * F[i * R + t];", "s += F[i * R + r] * F[i * R + r];", 0),
    ("frobenius_drops_square", "Table 2 Frobenius (P:176)",
     "s += H[i] * H[i];", "s += fabs(H[i]);", 0),
    ("objective_inner_product_factor", "Eq 6-7 (P:298-307)",
     "f[k] = xn2 - 2.0 * mdot + model_norm2(G[0], G[1], G[2], R);",
     "f[k] = xn2 - mdot + model_norm2(G[0], G[1], G[2], R);", 0),
    ("layout_key_a_b_swapped", "Table 2 (P:164-166), reading L1",
     "kv[e].key = (in * (uint64_t)dims[a] + ia) * (uint64_t)dims[b] + ib;",
     "kv[e].key = (in * (uint64_t)dims[b] + ib) * (uint64_t)dims[a] + ia;", 0),
    ("layout_duplicates_accepted", "S:108",
     "if (kv[e].key == kv[e - 1].key) { free(kv); return ORA_EDUP; }", "(void)0;", 0),
    ("init_wrong_bits", "C12",
     "F[n][i * R + r] = (double)(x >> 40) * (1.0 / 16777216.0);",
     "F[n][i * R + r] = (double)((x >> 16) & 0xFFFFFF) * (1.0 / 16777216.0);", 0),
    ("predict_drops_w", "Eq 8 (P:310)",
     "    for (int r = 0; r < R; r++)\n      xh += U[(int64_t)coords[3 * e] * R + r] * V[(int64_t)coords[3 * e + 1] * R + r] *\n            W[(int64_t)coords[3 * e + 2] * R + r];\n    out[e] = xh;",
     "    for (int r = 0; r < R; r++)\n      xh += U[(int64_t)coords[3 * e] * R + r] * V[(int64_t)coords[3 * e + 1] * R + r];\n    out[e] = xh;", 0),
    ("rmse_wrong_mean", "Eq 30 (P:886-890)",
     "sqrt(se / (double)n)", "sqrt(se / (double)(n + 1))", 0),
]


def _mutate(src, old, new, occ):
    pos = -1
    for _ in range(occ + 1):
        pos = src.find(old, pos + 1)
        assert pos >= 0, f"mutation anchor not found: {old!r}"
    return src[:pos] + new + src[pos + len(old):]


def _run_one(tmp, m):
    name, cite, old, new, occ = m
    mutated = _mutate(open(SRC).read(), old, new, occ)
    ms = os.path.join(tmp, f"{name}.c")
    with open(ms, "w") as fh:
        fh.write(mutated)
    env = dict(os.environ, ORACLE_SRC=ms, ORACLE_LIB=os.path.join(tmp, f"lib{name}.so"), OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_oracle_pins.py"), "-x",
                        "-q", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    return r.returncode, r.stdout[-2000:]


@pytest.fixture(scope="module")
def mutation_results(tmp_path_factory):
    """Every mutation's pin run, in parallel subprocesses (the suite stays within minutes)."""
    from concurrent.futures import ThreadPoolExecutor
    tmp = str(tmp_path_factory.mktemp("oracle_mutations"))
    with ThreadPoolExecutor(max_workers=max(2, min(16, (os.cpu_count() or 2)))) as ex:
        res = list(ex.map(lambda m: _run_one(tmp, m), MUTATIONS + [CONTROL]))
    return {m[0]: r for m, r in zip(MUTATIONS + [CONTROL], res)}


# the unmutated source through the same harness: must pass (the harness itself works)
CONTROL = ("control_unmutated", "-", "#include <math.h>", "#include <math.h>", 0)


def test_harness_control_passes(mutation_results):
    rc, out = mutation_results[CONTROL[0]]
    assert rc == 0, out


@pytest.mark.parametrize("name,cite", [(m[0], m[1]) for m in MUTATIONS], ids=[m[0] for m in MUTATIONS])
def test_pins_catch_mutation(mutation_results, name, cite):
    rc, out = mutation_results[name]
    assert rc != 0, f"mutation {name} ({cite}) survived every pin:\n{out}"
