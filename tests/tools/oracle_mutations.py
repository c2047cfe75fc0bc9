"""Mutation check of the oracle pins (run by hand: ``python tests/tools/oracle_mutations.py``).

Each mutation is a plausible slip in oracle/shiftk_oracle.c (dropped term, wrong sign, wrong
index, conjugation, transposed operand).  For each one the oracle is rebuilt and
tests/test_oracle_pins.py must FAIL.  The original source is always restored.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SRC = os.path.join(ROOT, "oracle", "shiftk_oracle.c")

MUTATIONS = [
    ("- c * ro[i]", "+ c * ro[i]"),                                       # sign, EQ-CG-RN-3REC
    ("rat * rat * beta", "rat * beta"),                                   # EQ-SHIFTEDCG-beta square
    ("- w - gamma * rho", "- w"),                                         # EQ-REC-ALPHA-N2 term
    ("- c * st->pi_old[k];", ";"),                                        # EQ-SHIFTEDCG-PI term
    ("*u = st->g[l] / st->pi[k]", "*u = st->g[l] / pin"),                # P:L373 index
    ("acc += 0.25 * J * r[s];", "acc += 0.5 * J * r[s];"),               # S^zS^z factor
    ("(1.0 + cc) * tn[i] - ac", "(1.0 + c) * tn[i] - ac"),               # BiCG shadow conj
    ("st->rho_prev /= fp * fp;", "st->rho_prev /= fp;"),                 # switch transform
    ("st->alpha_prev *= fp / f;", "st->alpha_prev *= f / fp;"),          # switch transform
    ("OR_COCG ? dot_plain(st, u, v)", "OR_COCG ? dot_conj(st, u, v)"),   # COCG inner product
    ("acc += 0.5 * J * r[s2];", "acc += 0.5 * J * r[s];"),               # flip partner
    ("int j = (i + 1) % L;", "int j = (i + 1 < L) ? i + 1 : i;"),        # periodic bond
    ("g[l] = dot_conj(st, st->left + l * st->M, v)",
     "g[l] = dot_plain(st, st->left + l * st->M, v)"),                    # a^dagger projection
    ("if (rank >= below) {", "if (rank > below) {"),                     # sector unrank
    ("rank += or_sz_dim(p, m);", "rank += or_sz_dim(p, m - 1);"),        # sector rank
    ("acc += 0.25 * J * r[a];", "acc += 0.25 * J * r[s];"),              # sector row vs state
    # row routines (the checkers of the sampled full-size GPU rows)
    ("acc += 0.5 * J * r[s ^ flip];", "acc += 0.5 * J * r[s ^ ((int64_t)1 << i)];"),   # row flip partner
    ("const int j = (i + 1) % L;                    /* bond", "const int j = (i + 1 < L) ? i + 1 : i; /* bond"),
    ("acc += val[e] * r[col[e]];      /* real row */", "acc += val[e] * r[i];      /* real row */"),  # CSR gather
    ("acc += val[e] * r[col[e]];      /* complex row */", "acc += conj(val[e]) * r[col[e]];      /* complex row */"),
    # the chunked fixed-order reduction and the in-place three-term update
    ("for (int64_t c = 0; c < nc; ++c) acc += part[c];", "for (int64_t c = 0; c + 1 < nc; ++c) acc += part[c];"),
    ("? i0 + OR_CHUNK : M;", "? i0 + OR_CHUNK - 1 : M;"),
    ("st->r = ro; st->r_old = rn;", "st->r = ro; st->r_old = ro;"),
    # contour-integral eigensolver (oracle/ss.py)
    ("s += (z[j] - gamma) / n_z * (z[j] - gamma) ** k * X[l, j]",
     "s += 1.0 / n_z * (z[j] - gamma) ** k * X[l, j]", "ss.py"),        # dz weight
    ("s += (z[j] - gamma) / n_z * (z[j] - gamma) ** k * X[l, j]",
     "s += (z[j] - gamma) / n_z * (z[j] - gamma) ** (k + 1) * X[l, j]", "ss.py"),   # moment order
    ("Ht = Ut.conj().T @ HU", "Ht = Ut.T @ HU", "ss.py"),               # Rayleigh-Ritz conj
]


def main():
    survived = []
    only = os.environ.get("MUTATIONS_ONLY")   # e.g. "ss.py": just the mutations of that file
    for m in MUTATIONS:
        if only and (m[2] if len(m) > 2 else "shiftk_oracle.c") != only:
            continue
        a, b = m[0], m[1]
        src = os.path.join(ROOT, "oracle", m[2]) if len(m) > 2 else SRC
        orig = open(src).read()
        assert a in orig, a
        try:
            open(src, "w").write(orig.replace(a, b, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q",
                                os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                               cwd=ROOT, capture_output=True, text=True)
            caught = r.returncode != 0
            print(("caught   " if caught else "SURVIVED ") + a + "  ->  " + b, flush=True)
            if not caught:
                survived.append(a)
        finally:
            open(src, "w").write(orig)
            os.utime(src)
    sys.exit(1 if survived else 0)


if __name__ == "__main__":
    main()
