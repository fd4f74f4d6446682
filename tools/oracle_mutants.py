"""Mutation check of the oracle's pins (VERDICT r01 "Next round" item 1).

Each mutant is a plausible mistake in oracle/loctomo_oracle.c; it is compiled
to /tmp and the -m "not gpu" pin suite (tests/test_oracle_pins.py) is run
against it through LT_ORACLE_SO.  A pinned oracle must fail at least one pin
for every mutant.  Usage: python tools/oracle_mutants.py [out.txt]
"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "loctomo_oracle.c")

# (name, old, new, expected occurrence count)
MUTANTS = [
    ("y forward projection: row/col offsets swapped (local_one)",
     "fp_rect(n, na, nd, ang, y, Wd, er0, ec0, H, Wd, sino);",
     "fp_rect(n, na, nd, ang, y, Wd, ec0, er0, H, Wd, sino);", 1),
    ("y backprojection: row/col offsets swapped (local_one)",
     "bp_rect(n, na, nd, ang, sino, g2, Wd, er0, ec0, H, Wd);",
     "bp_rect(n, na, nd, ang, sino, g2, Wd, ec0, er0, H, Wd);", 1),
    ("FISTA beta = (t'-1)/(t'+1) (local_one and or_global_tv)",
     "const double beta = momentum ? (t - 1.0) / tn : 0.0;",
     "const double beta = momentum ? (tn - 1.0) / (tn + 1.0) : 0.0;", 2),
    ("FISTA t update without the square (the paper's garbled line, P:L679)",
     "const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); /* A12 */",
     "const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t)); /* A12 */", 1),
    ("FISTA beta uses t_k instead of t_{k-1} (local_one and or_global_tv)",
     "const double beta = momentum ? (t - 1.0) / tn : 0.0;",
     "const double beta = momentum ? (tn - 1.0) / tn : 0.0;", 2),
    ("FGP inner momentum beta = (t'-1)/(t'+1)",
     "const double beta = (t - 1.0) / tn;",
     "const double beta = (tn - 1.0) / (tn + 1.0);", 1),
    ("disc term dropped from x_s",
     "if (xx * xx + yy * yy <= rad2) xs[(size_t)i * Wd + j] += discc;",
     "if (xx * xx + yy * yy <= rad2) xs[(size_t)i * Wd + j] += 0.0 * discc;", 1),
    ("box update keeps y = S - x_s (no clamp correction d)",
     "y[e] = x[e] - xs[e];",
     "y[e] = s - xs[e];", 1),
    ("x_s from b_{k+1} (filter index off by one)",
     "bp_rect(n, na, nd, ang, bconv + (size_t)k * ns, xs, Wd, er0, ec0, H, Wd);",
     "bp_rect(n, na, nd, ang, bconv + (size_t)(k + 1 < nk ? k + 1 : k) * ns, xs, Wd, er0, ec0, H, Wd);", 1),
    ("projector weight missing the 1/c factor",
     "row[d] += hat((d - tau) / c) / c * v;",
     "row[d] += hat((d - tau) / c) * v;", 1),
]


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    src = open(SRC).read()
    lines = []
    survivors = 0
    with tempfile.TemporaryDirectory() as td:
        for i, (name, old, new, cnt) in enumerate(MUTANTS):
            got = src.count(old)
            assert got == cnt, (name, got)
            mfile = os.path.join(td, f"m{i}.c")
            so = os.path.join(td, f"m{i}.so")
            open(mfile, "w").write(src.replace(old, new))
            subprocess.check_call(["gcc", "-O2", "-msse4.1", "-std=gnu11", "-fopenmp", "-fPIC", "-shared",
                                   "-fno-fast-math", mfile, "-o", so, "-lm"])
            env = dict(os.environ, LT_ORACLE_SO=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                                os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            failed = sorted(set(re.findall(r"FAILED tests/test_oracle_pins.py::(\S+)", r.stdout)))
            summ = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else "?"
            killed = r.returncode != 0 and failed
            survivors += 0 if killed else 1
            lines.append(f"[{'KILLED' if killed else 'SURVIVED'}] {name}\n    {summ}\n    failing pins: "
                         + (", ".join(failed) if failed else "-"))
            print(lines[-1], flush=True)
    lines.append(f"\n{len(MUTANTS) - survivors}/{len(MUTANTS)} mutants killed by tests/test_oracle_pins.py")
    print(lines[-1])
    if out_path:
        with open(out_path, "w") as f:
            f.write("# oracle mutation check: python tools/oracle_mutants.py (each mutant = one edit of "
                    "oracle/loctomo_oracle.c, pin suite run against it)\n")
            f.write("\n".join(lines) + "\n")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
