#!/usr/bin/env python
"""The paper's numerical verification of RBM-1 (Sec. 4.1) on
the GPU, against the GPU direct O(N^2) step (row f1):

  Fig. errdepN  E^(T=1) vs tau in {2^-4..2^-7}, N in {50, 500, 2000}, beta in {0, 1}
  Fig. errdepT  E^(T) vs T for tau = 2^-7, N = 500, beta in {0, 1}
  Fig. cpu      error vs device time, RBM-1 vs direct forward Euler, N in {1e3, 1e4}

E^(T) = sqrt(mean_i |X_rbm^i(T) - X_ref^i(T)|^2) (Eq. 4.2); the reference
is the fully coupled forward Euler solution with tau = 2^-15; X_0 iid
from rho_0 = sqrt(4-x^2)/(2 pi); smooth test system K(x) = x/(1+x^2),
V = beta x^2/2, sigma = 0.  Writes a JSON + markdown table.

    python scripts/convergence_study.py [--out profiles/r1b_convergence]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import rbm_inputs as RI  # noqa: E402
from paper_1812_10575_b200 import RBM, Direct  # noqa: E402


def system(n, beta, seed, dt, dtype="f64"):
    return dict(RI.smooth_test(n, p=2, beta=beta, seed=seed, dtype=dtype), sigma=0.0, init="user", dt=dt)


def reference(n, beta, seed, T, exp=15):
    x0 = RI.semicircle_x0(n, seed=seed)
    d = Direct(system(n, beta, seed, 2.0 ** -exp), x0)
    d.run(int(round(T * 2 ** exp)))
    return x0, d.gather()


def rbm(x0, n, beta, seed, T, exp):
    s = RBM(system(n, beta, seed, 2.0 ** -exp), x0=x0)
    s.run(int(round(T * 2 ** exp)))
    x = s.gather(host=True)
    s.close()
    return x


def err(a, b):
    return float(np.sqrt(np.mean((np.asarray(a) - np.asarray(b)) ** 2)))


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1b_convergence"))
    args = ap.parse_args()
    res = {"errdepN": [], "errdepT": [], "cpu": []}
    for beta in (0.0, 1.0):
        for n in (50, 500, 2000):
            x0, ref = reference(n, beta, seed=1, T=1.0)
            row = {"beta": beta, "N": n, "tau_exp": [], "E": []}
            for k in (4, 5, 6, 7):
                row["tau_exp"].append(k)
                row["E"].append(err(rbm(x0, n, beta, 1, 1.0, k), ref))
            row["slope"] = float(np.polyfit(np.log([2.0 ** -k for k in row["tau_exp"]]), np.log(row["E"]), 1)[0])
            res["errdepN"].append(row)
    for beta in (0.0, 1.0):
        row = {"beta": beta, "N": 500, "T": [], "E": []}
        for T in (0.5, 1.0, 2.0, 4.0):
            x0, ref = reference(500, beta, seed=2, T=T)
            row["T"].append(T)
            row["E"].append(err(rbm(x0, 500, beta, 2, T, 7), ref))
        res["errdepT"].append(row)
    # error vs device time (Fig. cpu): both methods with tau = 2^-1 .. 2^-6
    for n in (1000, 10000):
        x0, ref = reference(n, 1.0, seed=3, T=1.0, exp=12 if n > 1000 else 15)
        for k in (1, 2, 3, 4, 5, 6):
            cfg = system(n, 1.0, 3, 2.0 ** -k)
            s = RBM(cfg, x0=x0)
            _, t_rbm = timed(lambda: s.run(2 ** k))
            e_rbm = err(s.gather(host=True), ref)
            s.close()
            d = Direct(cfg, x0)
            _, t_dir = timed(lambda: d.run(2 ** k))
            e_dir = err(d.gather(), ref)
            res["cpu"].append({"N": n, "tau_exp": k, "rbm_s": t_rbm, "rbm_E": e_rbm, "direct_s": t_dir,
                               "direct_E": e_dir})
    with open(args.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = ["# RBM-1 convergence study on B200 (paper Sec. 4.1; `scripts/convergence_study.py`)", "",
             "Smooth test system K(x)=x/(1+x^2), V=beta x^2/2, sigma=0; X_0 iid semicircle on [-2,2];",
             "reference = GPU direct forward Euler with tau=2^-15; RBM-1 with p=2.", "",
             "## E^(T=1) vs tau (Fig. errdepN)", "", "| beta | N | tau=2^-4 | 2^-5 | 2^-6 | 2^-7 | slope |",
             "|---|---|---|---|---|---|---|"]
    for r in res["errdepN"]:
        lines.append(f"| {r['beta']:g} | {r['N']} | " + " | ".join(f"{e:.3e}" for e in r["E"]) + f" | {r['slope']:.2f} |")
    lines += ["", "## E^(T) vs T, tau = 2^-7, N = 500 (Fig. errdepT)", "", "| beta | T=0.5 | 1 | 2 | 4 |", "|---|---|---|---|---|"]
    for r in res["errdepT"]:
        lines.append(f"| {r['beta']:g} | " + " | ".join(f"{e:.3e}" for e in r["E"]) + " |")
    lines += ["", "## Error vs wall time, beta = 1, T = 1 (Fig. cpu; device-synchronised wall clock)", "",
              "| N | tau | RBM-1 s | RBM-1 E^ | direct s | direct E^ |", "|---|---|---|---|---|---|"]
    for r in res["cpu"]:
        lines.append(f"| {r['N']} | 2^-{r['tau_exp']} | {r['rbm_s']:.4f} | {r['rbm_E']:.3e} | {r['direct_s']:.4f} | {r['direct_E']:.3e} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
