"""Mutation check of the oracle's pins (VERDICT r1 Weak #1): apply one plausible
transcription error at a time to a scratch copy of oracle/chemora_oracle.cpp and run the
CPU oracle pins (tests/test_oracle_*.py) against it; every mutation must make at least one
pin fail.  Usage: python scripts/oracle_mutations.py [test-file ...] [> profiles/r2_oracle_mutations.txt]
(with test files given, only those pins run -- e.g. the behavioural gauge pins alone)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTATIONS = [
    ("drop c_alpha_adv Adv(A) in d_t A", "+ P.c_alpha_adv * adv(AUXA)", ""),
    ("flip the sign of -Adv(Xt) in d_t B", "(adv(BB + i) - adv(XT + i))", "(adv(BB + i) + adv(XT + i))"),
    ("drop Adv(B) in d_t B", "(adv(BB + i) - adv(XT + i))", "(-adv(XT + i))"),
    ("flip the sign of eta beta in the (1 - S_B) branch", "(Xt[i] - P.eta * beta[i])", "(Xt[i] + P.eta * beta[i])"),
    ("change the exponent p_beta", "std::pow(alpha, P.p_beta)", "std::pow(alpha, P.p_beta + 1.0)"),
    ("change the exponent n_alpha", "std::pow(alpha, P.n_alpha)", "std::pow(alpha, P.n_alpha - 1.0)"),
    ("(1 - L) K -> (1 - L) A in d_t alpha", "(1.0 - P.L) * trK)", "(1.0 - P.L) * Aux)"),
    ("drop S_B in d_t B", "P.S_B * (rhs_Xt[i] - P.eta * B[i])", "(rhs_Xt[i] - P.eta * B[i])"),
    ("control: B damping x2", "P.S_B * (rhs_Xt[i] - P.eta * B[i])", "P.S_B * (rhs_Xt[i] - 2.0 * P.eta * B[i])"),
    ("drop Xtn (Gl + Gl) in the Ricci tensor", "for (int kx = 0; kx < 3; ++kx) r += 0.5 * Xtn[kx] * (Gl[i][j][kx] + Gl[j][i][kx]);\n            for (int l = 0; l < 3; ++l)\n              for (int m = 0; m < 3; ++m)\n                for (int kx = 0; kx < 3; ++kx)\n                  r += gu[l][m] * (Gu[kx][l][i] * Gl[j][kx][m] + Gu[kx][l][j] * Gl[i][kx][m] +\n                                   Gu[kx][i][m] * Gl[kx][l][j]);\n            Rt[i][j] = r;",
     "for (int l = 0; l < 3; ++l)\n              for (int m = 0; m < 3; ++m)\n                for (int kx = 0; kx < 3; ++kx)\n                  r += gu[l][m] * (Gu[kx][l][i] * Gl[j][kx][m] + Gu[kx][l][j] * Gl[i][kx][m] +\n                                   Gu[kx][i][m] * Gl[kx][l][j]);\n            Rt[i][j] = r;"),
    ("conformal factor of the physical Christoffel: 2 -> 1", "gphys += 2.0 * corr;", "gphys += corr;"),
    ("K^2/3 -> K^2/2 in d_t K", "alpha * (AA + trK * trK / 3.0)", "alpha * (AA + trK * trK / 2.0)"),
    ("6 At^ij d_j phi -> 5 in d_t Xt", "s += 6.0 * Atu[i][j] * dphi[j];", "s += 5.0 * Atu[i][j] * dphi[j];"),
    ("1/3 -> 1/2 of gt^ij d_j(div beta) in d_t Xt", "r += gu[i][j] * ddivbeta[j] / 3.0;", "r += gu[i][j] * ddivbeta[j] / 2.0;"),
    ("transpose dbeta in d_t gt", "r += gt[i][kx] * dbeta[j][kx] + gt[j][kx] * dbeta[i][kx];", "r += gt[i][kx] * dbeta[kx][j] + gt[j][kx] * dbeta[kx][i];"),
    ("drop Gt^j_jk At^ik in the momentum constraint", "for (int kx = 0; kx < 3; ++kx) m += Gu[j][j][kx] * Atu[i][kx];", ""),
    ("upwind: swap D+ and D-", "s += bp * dplus(F(v), c, st[l], h[l]) + bm * dminus(F(v), c, st[l], h[l]);",
     "s += bp * dminus(F(v), c, st[l], h[l]) + bm * dplus(F(v), c, st[l], h[l]);"),
]


def main():
    src = open(os.path.join(ROOT, "oracle", "chemora_oracle.cpp")).read()
    tests = sys.argv[1:] or sorted(f for f in os.listdir(os.path.join(ROOT, "tests")) if f.startswith("test_oracle_"))
    ok = True
    for name, old, new in MUTATIONS:
        if src.count(old) < 1:
            print(f"SKIP (pattern not found): {name}")
            ok = False
            continue
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "chemora_inputs"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            with open(os.path.join(tmp, "oracle", "chemora_oracle.cpp"), "w") as fh:
                fh.write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                *[os.path.join("tests", t) for t in tests]], cwd=tmp,
                               capture_output=True, text=True, timeout=900)
            failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            caught = r.returncode != 0
            ok = ok and caught
            print(f"{'caught' if caught else 'MISSED'}: {name}" + (f"  <- {failed[0]}" if failed else ""), flush=True)
    print("all mutations caught" if ok else "SOME MUTATIONS MISSED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
