"""Writes tests/golden/fista_tk.txt: the FISTA step-size sequence of Beck &
Teboulle (2009), the method Alg. 3 of the paper follows ("we use similar
notation to [Beck2009a]"; Alg. 3, garbled there --
reading A12 in DESIGN.md):

    t_1 = 1,  t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2,
    momentum after the k-th prox step  beta_k = (t_k - 1) / t_{k+1}.

Computed with Python's decimal module at 50 significant digits (no oracle, no
CUDA path).  tests/test_oracle_pins.py checks the table against properties the
sequence must have (t_2 = the golden ratio, t_{k+1}^2 - t_{k+1} = t_k^2,
t_k >= (k+1)/2) before using it to pin the oracle's momentum step.
Run: python tests/golden/make_fista_tk.py
"""
import os
from decimal import Decimal, getcontext

getcontext().prec = 50
K = 60
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fista_tk.txt")
t = Decimal(1)
rows = []
for k in range(1, K + 1):
    tn = (1 + (1 + 4 * t * t).sqrt()) / 2
    rows.append((k, t, (t - 1) / tn))
    t = tn
with open(out, "w") as f:
    f.write("# FISTA sequence (Beck & Teboulle 2009; PAPER.md L660, Alg. 3 L679-680 per reading A12)\n")
    f.write("# k  t_k  beta_k = (t_k - 1) / t_{k+1}   -- written by tests/golden/make_fista_tk.py\n")
    for k, tk, bk in rows:
        f.write(f"{k} {tk:.30e} " + (f"{bk:.30e}" if bk else "0.0") + "\n")
