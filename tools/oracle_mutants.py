"""Mutation check of the oracle pins (CPU only; not part of the product or the test suite).

Each mutant is one plausible mistake in oracle/hh_ref.c (a dropped factor, a wrong sign,
a transposed operand, a swapped order, a tie rule).  The tool applies it to the source,
rebuilds libhh_ref.so, runs tests/test_oracle_pins.py and reports whether a pin failed
("killed").  A surviving mutant means a pin is missing.  The source is restored afterwards.

usage: python tools/oracle_mutants.py [substring-of-mutant-name ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "hh_ref.c")

# (name, old text, new text, which occurrence of `old` (0-based) to replace)
MUTANTS = [
    ("reflect: factor 2 dropped", "a = 2.0 * a;", "a = 1.0 * a;", 0),
    ("reflect: update sign", "x[r] -= a * u[r];", "x[r] += a * u[r];", 0),
    ("reflect: dot uses x*x", "a += u[r] * x[r];", "a += x[r] * x[r];", 0),
    ("apply_one: order of op N / op T swapped", "if (op == 0) {\n        for (int64_t i = h - 1",
     "if (op == 1) {\n        for (int64_t i = h - 1", 0),
    ("apply_one: op N skips the last reflector", "for (int64_t i = h - 1; i >= 0; --i)",
     "for (int64_t i = h - 2; i >= 0; --i)", 0),
    ("sym: Q pass first (transposed)", "apply_one(1, n, h, U, x);\n                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];\n                apply_one(0, n, h, U, x);\n                memcpy",
     "apply_one(0, n, h, U, x);\n                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];\n                apply_one(1, n, h, U, x);\n                memcpy", 0),
    ("sym: lambda dropped", "for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];\n                apply_one(0, n, h, U, x);\n                memcpy",
     "apply_one(0, n, h, U, x);\n                memcpy", 0),
    ("mahalanobis: sum instead of difference", "z[r] = xa[r] - xb[r];", "z[r] = xa[r] + xb[r];", 0),
    ("mahalanobis: Q instead of Q^T", "apply_one(1, n, h, U, z);\n                double s = 0.0;",
     "apply_one(0, n, h, U, z);\n                double s = 0.0;", 0),
    ("mahalanobis: d dropped", "s += d[r] * (z[r] * z[r]);", "s += (z[r] * z[r]);", 0),
    ("mahalanobis: d squared", "s += d[r] * (z[r] * z[r]);", "s += d[r] * d[r] * (z[r] * z[r]);", 0),
    ("apply_signed: sides swapped", "if (side == 1)\n                    for (int64_t r = 0; r < n; ++r) x[r] *= d[r];",
     "if (side == 0)\n                    for (int64_t r = 0; r < n; ++r) x[r] *= d[r];", 0),
    ("sym_signed: trailing D dropped", "apply_one(0, n, h, U, x);\n                for (int64_t r = 0; r < n; ++r) x[r] *= d[r];\n",
     "apply_one(0, n, h, U, x);\n", 0),
    ("sym_signed: leading D dropped", "for (int64_t r = 0; r < n; ++r) x[r] *= d[r];\n                apply_one(1, n, h, U, x);\n                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];",
     "apply_one(1, n, h, U, x);\n                for (int64_t r = 0; r < n; ++r) x[r] *= lam[r];", 0),
    ("knn: later index wins ties (skip rule)", "!(s < bd[k - 1])", "(s > bd[k - 1])", 0),
    ("knn: later index wins ties (insertion)", "bd[pos - 1] > s", "bd[pos - 1] >= s", 0),
    ("knn: Q instead of Q^T", "apply_one(1, n, h, U, z);\n                    double s = 0.0;",
     "apply_one(0, n, h, U, z);\n                    double s = 0.0;", 0),
    ("knn: d dropped", "s += d[e] * (z[e] * z[e]);", "s += (z[e] * z[e]);", 0),
    ("congruence: second apply on the untransposed matrix", "rc = hh_ref_apply(op, n, h, U, B, A, n);",
     "rc = hh_ref_apply(op, n, h, U, A, B, n), memcpy(A, B, sizeof(double) * nn);", 0),
    ("congruence: second apply with the other op", "rc = hh_ref_apply(op, n, h, U, B, A, n);",
     "rc = hh_ref_apply(1 - op, n, h, U, B, A, n);", 0),
    ("shf: cost factor", "cost[k] = q - 2.0 * (qa * qb);", "cost[k] = q - 4.0 * (qa * qb);", 0),
    ("shf: cost sign", "cost[k] = q - 2.0 * (qa * qb);", "cost[k] = q + 2.0 * (qa * qb);", 0),
    ("shf: BA term dropped", "for (int64_t l = 0; l < n; ++l) s += B[i * n + l] * A[l * n + j];", "", 0),
    ("shf: gradient factor", "g[i] = 2.0 * mi - 4.0 * ci;", "g[i] = 2.0 * mi - 2.0 * ci;", 0),
    ("shf: gradient A / B swapped", "ci += (qa * B[i * n + j] + qb * A[i * n + j]) * u[j];",
     "ci += (qa * A[i * n + j] + qb * B[i * n + j]) * u[j];", 0),
]


def nth_replace(text, old, new, k):
    pos = -1
    for _ in range(k + 1):
        pos = text.find(old, pos + 1)
        if pos < 0:
            raise ValueError(f"pattern not found: {old[:50]!r}")
    return text[:pos] + new + text[pos + len(old):]


def run_pins():
    env = dict(os.environ, OMP_NUM_THREADS="8")
    p = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q",
                        "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True)
    tail = [l for l in p.stdout.splitlines() if l.startswith("FAILED") or " passed" in l or " failed" in l]
    return p.returncode, tail


def main():
    want = sys.argv[1:]
    orig = open(SRC).read()
    survivors = []
    try:
        for name, old, new, k in MUTANTS:
            if want and not any(w in name for w in want):
                continue
            open(SRC, "w").write(nth_replace(orig, old, new, k))
            rc, tail = run_pins()
            killed = rc != 0
            print(f"{'killed  ' if killed else 'SURVIVED'}  {name}  {tail[:1]}", flush=True)
            if not killed:
                survivors.append(name)
    finally:
        open(SRC, "w").write(orig)
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT)
    print(f"{len(survivors)} survivor(s): {survivors}")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
