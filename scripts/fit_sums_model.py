"""Fit the plan cost model's constants for the sum-plane 3M kernels (cfg 14, 15) to
filter-call sweeps (scripts/probe_sums.py with SUMS_ONLY=1; profiles/r01/sweep_sums_*.json).

    python scripts/fit_sums_model.py profiles/r01/sweep_sums_20000.json [...]

Same model form as csrc/zgemm.cu `plan_cost` (scripts/fit_cost_model.py), with its own
efficiencies, ragged-tile floor / imbalance, pipe-sharing constant and split-K reduce
cost for these kernels (3 CTAs per SM). Prints the constants and, per shape, the
measured speed of the model's pick against the best measured plan.
"""
import json
import math
import sys

import numpy as np
from scipy.optimize import least_squares

BM, BN = 64, 32
WN = {14: 16, 15: 32}
OCC = 3
SMS = 148
PEAK = 37.16e12 / 8.0 / 1e6 / SMS  # complex MACs per microsecond per SM at the DMMA peak
HBM = 6.58e6  # bytes per microsecond


def model(p, n, k, c, s):
    eff14, eff15, r0, floor, rag, t0, tred = p
    eff = eff14 if c == 14 else eff15
    M = K = n
    tm = -(-M // BM)
    tn = -(-k // BN)
    ctas = tm * tn * s
    q = -(-ctas // SMS)
    kchunk = -(-K // s)
    last = -(-(k - (tn - 1) * BN) // 8) * 8
    live = ((tn - 1) * BN + max(last, floor * BN)) / tn
    W = BM * live * kchunk
    full, rem = divmod(q, OCC)
    rounds = full * max(OCC, r0) + (max(rem, r0) if rem else 0.0)
    t = W * rounds / (eff * PEAK)
    per, wcols = WN[c] // 8, BN // WN[c]
    vb = last // 8
    lives = [max(0, min(per, vb - w * per)) for w in range(wcols)]
    if max(lives) != min(lives):
        t *= 1.0 + rag / tn
    t += t0
    if s > 1:
        t += tred + (s + 3) * M * k * 16.0 / HBM
    return t


def main():
    rows = []
    for path in sys.argv[1:]:
        d = json.load(open(path))
        n = d["n"]
        for k, r in d["widths"].items():
            k = int(k)
            for key, tf in r.items():
                if not key.startswith("c"):
                    continue
                c, s = key[1:].split("s")
                us = 8.0 * n * n * k / (tf * 1e12) * 1e6
                rows.append((n, k, int(c), int(s), us))
    p0 = [1.25, 1.25, 1.3, 0.86, 0.12, 5.0, 3.0]

    def resid(p):
        return [math.log(model(p, n, k, c, s) / us) for n, k, c, s, us in rows]

    fit = least_squares(resid, p0, bounds=([0.5, 0.5, 1.0, 0.0, 0.0, 0.0, 0.0],
                                           [2.0, 2.0, 3.0, 1.0, 2.0, 100.0, 100.0]))
    print("eff14 eff15 r0 floor rag t0 tred =", [round(x, 4) for x in fit.x])
    shapes = {}
    for n, k, c, s, us in rows:
        shapes.setdefault((n, k), []).append((c, s, us))
    losses = []
    for (n, k), cand in sorted(shapes.items()):
        best = min(cand, key=lambda x: x[2])
        pick = min(cand, key=lambda x: model(fit.x, n, k, x[0], x[1]))
        losses.append(pick[2] / best[2])
        print(f"n={n} k={k}: pick c{pick[0]}s{pick[1]} {pick[2] / best[2]:.3f} of best "
              f"(best c{best[0]}s{best[1]})")
    print("geomean pick/best", float(np.exp(np.mean(np.log(losses)))), "max", max(losses))


if __name__ == "__main__":
    main()
