"""Per-rank cost of one column-sharded outer iteration at N = 1, 2, 4, 8, measured on
one B200 (the work one rank does in distributed.ShardedPhases; no rank waits on
another, so nothing here needs the other GPUs):

  filter      m fused degree steps on the rank's ceil(k/N)-column shard (H declared)
  project     CGS2 of the shard against the L locked vectors
  cholqr      2 passes: Gram X^H X[:, p] (k x k_p), replicated Cholesky + inverse of
              the gathered k x k Gram, X R^-1[:, p] (triangle-skipping)
  rr          H Q[:, p], Q^H HQ[:, p], replicated hermitize + zheevd(k), Z[:, p] and
              HZ[:, p] = Q W[:, p], HQ W[:, p], residual norms of the own columns
  guard       the cross-rank agreement all-gathers are tiny; their cost is in `gather`
  gather      NCCL all-gathers modelled at BUS_GBS per GPU: F, T, Q (n x k each),
              HQ (n x k), three k x k Grams, residuals, plus LAT_US per collective

Widths: the full block (k = 2200, no locked vectors: the first iterations) and the
reference-interval tail (k = 201 against L = 2000 locked: 5006 of the 5024 iterations
of the one-GPU c4 solve). The slowest rank holds ceil(k / N) columns.

    python scripts/rank_phase_probe.py > gpurun_out/rank_phases.json
"""
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

N_ORDER = 20000
DEGREE = 25
BUS_GBS = 600.0     # conservative NVLink 5 all-gather bus bandwidth per GPU
LAT_US = 30.0       # per-collective launch + sync latency
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
n = N_ORDER
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
H = ((H + H.T.conj()) * (0.5 / (3.0 * math.sqrt(n)))).resolve_conj().contiguous()  # |lambda| < 1
eng.declare_operator(H)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e-3 / reps


def probe(k, L, N):
    kp = -(-k // N)
    lo = 0
    X = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g) / math.sqrt(n)
    Xq = torch.linalg.qr(X.T)[0].T.contiguous()  # orthonormal k-column block (cols, rows)
    Y = X[:kp].clone() * 1e-3
    W = torch.empty_like(Y)
    Lk = None
    if L:
        Lk = torch.linalg.qr(torch.randn((n, L), dtype=torch.complex128, device=dev,
                                         generator=g))[0].T.contiguous()
    G = torch.empty((k, k), dtype=torch.complex128, device=dev)
    Gs = torch.empty((k, k), dtype=torch.complex128, device=dev)
    eng.zgemm("C", "N", k, k, n, 1.0, Xq, Xq, 0.0, Gs)  # SPD (identity-like) Gram
    Li = torch.empty_like(G)
    out_p = torch.empty((kp, n), dtype=torch.complex128, device=dev)
    HQ = torch.empty((k, n), dtype=torch.complex128, device=dev)
    eng.apply_operator(H, Xq, HQ)
    t = {}
    t["filter"] = timed(lambda: eng.filter(H, Y, W, DEGREE, -1.0, 1.0, -2.0), reps=2)
    t["project"] = timed(lambda: eng.project_out(out_p.copy_(X[:kp]), Lk)) if L else 0.0

    def gram():
        eng.zgemm("C", "N", k, kp, n, 1.0, Xq, Xq[lo:lo + kp], 0.0, G[lo:lo + kp])

    def chol():
        G.copy_(Gs)
        eng.cholesky_inverse(G, Li)

    def apply():
        eng.zgemm("N", "C", n, kp, k, 1.0, Xq, Li[:, lo:lo + kp], 0.0, out_p,
                  tri=eng.TRI_B_UPPER, tri_offset=lo)

    t["cholqr"] = 2 * (timed(gram) + timed(chol) + timed(apply))
    hq_p = HQ[:kp]

    def rr_dist():
        eng.apply_operator(H, Xq[:kp], hq_p)
        eng.zgemm("C", "N", k, kp, n, 1.0, Xq, hq_p, 0.0, G[:kp])

    def eig():
        G.copy_(Gs)
        eng.hermitize(G)
        eng.heevd(G)

    Wv = Gs.clone()

    def ritz():
        eng.zgemm("N", "N", n, kp, k, 1.0, Xq, Wv[:kp], 0.0, out_p)
        eng.zgemm("N", "N", n, kp, k, 1.0, HQ, Wv[:kp], 0.0, W[:kp])
        eng.residual_norms(W[:kp], out_p, np.zeros(kp))

    t["rr"] = timed(rr_dist) + timed(eig) + timed(ritz)
    if N > 1:
        nbytes = 16.0 * n * k * 4 + 16.0 * k * k * 3 + 8.0 * k
        t["gather"] = nbytes * (N - 1) / N / (BUS_GBS * 1e9) + 9 * LAT_US * 1e-6
    else:
        t["gather"] = 0.0
    t["total"] = sum(t.values())
    t["k"], t["L"], t["N"], t["shard"] = k, L, N, kp
    return t


rows = []
for (k, L) in ((2200, 0), (201, 2000)):
    for N in (1, 2, 4, 8):
        r = probe(k, L, N)
        rows.append(r)
        print(json.dumps({kk: (round(v, 5) if isinstance(v, float) else v) for kk, v in r.items()}),
              file=sys.stderr, flush=True)
eng.declare_operator(None)
summary = {}
for (k, L) in ((2200, 0), (201, 2000)):
    t1 = next(r["total"] for r in rows if r["k"] == k and r["N"] == 1)
    summary[f"k{k}_L{L}"] = {str(r["N"]): {"s_per_iteration": r["total"],
                                           "efficiency": t1 / (r["N"] * r["total"])}
                            for r in rows if r["k"] == k}
print(json.dumps({"n": n, "degree": DEGREE, "bus_gbs": BUS_GBS, "lat_us": LAT_US,
                  "rows": rows, "summary": summary}, indent=1))
