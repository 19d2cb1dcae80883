"""Strong-scaling model of a full ChFSI solve on N GPUs from 1-GPU measurements
(this run has one B200; the driver measures the filter bench at N = 1..8).

    python scripts/scaling_model.py SOLVE.json KXK.json [TUNE.json]

    e.g. SOLVE.json = profiles/r01/solves/c4_standard_problem1_block_top_3m.json
         (block_top) or ..._reference_interval_3m.json (the reference's semantics);
         KXK.json = profiles/r01/kxk_probe.json; TUNE.json defaults to the 3M
         per-width table profiles/r01/filter_widths_3m.json.

Inputs, all measured on one B200:
  SOLVE.json  scripts/c4_solve.py output with per-iteration phase times
              [cols, locked, t_filter, t_qr, t_rr] (1 GPU);
  KXK.json    scripts/kxk_probe.py: replicated k x k step times (Cholesky + inverse
              per CholQR pass, hermitize + zheevd per Rayleigh-Ritz);
  TUNE.json   scripts/tune_sweep.py filter-step timings (planner picks, "cfg": -1)
              at n = 20000, for the filter speed of a k/N-column shard.
Per iteration of width k on N ranks (distributed.ShardedPhases):
  filter     m * t_step(ceil(k / N))                      (shard width speed)
  QR         (t_qr - 2 chol(k)) / N + 2 chol(k)           (n-sized GEMMs sharded)
  RR         (t_rr - eig(k)) / N + eig(k)                 (HQ, Gram, Z/HZ sharded)
  gathers    4 n k 16 B + 3 k^2 16 B over NVLink at BW (F, T, Q, HQ; 3 Grams)
and, for comparison, the first multi-GPU version that replicated QR and all of RR
except HQ. Setup (Lanczos, bootstrap, final re-check) is taken as sharded like RR.
"""
import json
import math
import sys


N_ORDER = 20000
DEGREE = 25
NVLINK_BPS = 600e9  # conservative all-gather bus bandwidth per GPU


def interp(table, k):
    ks = sorted(table)
    if k <= ks[0]:
        return table[ks[0]] * k / ks[0]
    if k >= ks[-1]:
        return table[ks[-1]] * k / ks[-1]
    for a, b in zip(ks, ks[1:]):
        if a <= k <= b:
            t = (math.log(k) - math.log(a)) / (math.log(b) - math.log(a))
            return math.exp((1 - t) * math.log(table[a]) + t * math.log(table[b]))
    raise ValueError(k)


def main():
    solve = json.load(open(sys.argv[1]))
    kxk = {int(k): v for k, v in json.load(open(sys.argv[2])).items()}
    tune_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/r01/filter_widths_3m.json"
    step = {r["k"]: r["ms"] * 1e-3 for r in json.load(open(tune_path))
            if r["cfg"] == -1 and r["n"] == N_ORDER}
    chol = {k: v["chol_inv_s"] for k, v in kxk.items()}
    eig = {k: v["eig_s"] for k, v in kxk.items()}
    p = solve["problems"][0]
    its = p["iterations"]
    t1 = p["s_per_solve"]
    loop1 = sum(i[2] + i[3] + i[4] for i in its)
    setup1 = t1 - loop1
    print(f"1 GPU: {t1:.1f} s ({len(its)} iterations; filter {p['t_filter']:.1f}, "
          f"QR {p['t_qr']:.2f}, RR {p['t_rr']:.2f}, setup/other {setup1:.2f})")
    for ngpu in (2, 4, 8):
        # filter alone: the widest shard's padded DMMA work sets the time
        tf1 = sum(i[2] for i in its)
        tfn = sum(DEGREE * interp(step, -(-i[0] // ngpu)) for i in its if i[0])
        print(f"N={ngpu}: filter-only bound {tf1 / (ngpu * tfn):.3f} "
              f"(1-GPU filter {tf1:.1f} s, per-rank filter {tfn:.1f} s)")
        new = old = 0.0
        for cols, _, tf, tq, tr in its:
            kp = -(-cols // ngpu)
            tf_n = DEGREE * interp(step, kp) if kp else 0.0
            kk_chol = 2 * interp(chol, cols)
            kk_eig = interp(eig, cols)
            gather = (4 * N_ORDER * cols * 16 + 3 * cols * cols * 16) / NVLINK_BPS
            hq = tf / DEGREE
            new += (tf_n + max(tq - kk_chol, 0.0) / ngpu + kk_chol
                    + max(tr - kk_eig, 0.0) / ngpu + kk_eig + gather)
            old += tf_n + tq + hq / ngpu + (tr - hq) + 2 * 16 * N_ORDER * cols / NVLINK_BPS
        new += setup1 / ngpu
        old += setup1
        print(f"N={ngpu}: sharded QR/RR {new:7.2f} s (efficiency {t1 / (ngpu * new):.3f}); "
              f"replicated QR/RR {old:7.2f} s ({t1 / (ngpu * old):.3f})")


if __name__ == "__main__":
    main()
