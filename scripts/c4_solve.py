"""Full ChFSI solves at BASELINE c4 scale on one B200 (data generated on the device).

    python scripts/c4_solve.py [--n 20000] [--nev 2000] [--nex 200] [--degree 25]
                               [--interval block_top|reference] [--problems 1]
                               [--generalized] [--max-it 20000] [--out gpurun_out/c4.json]

Problem recipe (BASELINE c2-c4): A_1 with the c0 spectrum (H = Q diag Q^H), A_{i+1} =
A_i + delta E_i, E_i = (G+G^H)/2 scaled by a 10-step Lanczos estimate of ||E_i||_2,
delta = 1e-3 ||A_1||_2; S = I + 0.1 B^H B / ||B^H B|| (Lanczos estimate) when
--generalized. The sequence is solved with eigenvector reuse (solve_sequence
semantics). Verification: residuals, B-orthonormality, and for problem 1 (exact
spectrum known) the relative eigenvalue error of the standard problem.
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1305_5120_b200 as G  # noqa: E402
from paper_1305_5120_b200 import device as D  # noqa: E402
from paper_1305_5120_b200 import workloads as Wl  # noqa: E402


def lanczos_norm(eng, blk, seed):
    n = blk.shape[1]
    v = np.random.default_rng(seed).standard_normal(n) + 0j
    v /= np.linalg.norm(v)
    b, al, be = eng.lanczos_bound(blk, D.to_device(v, blk.device), 10)
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--nev", type=int, default=2000)
    ap.add_argument("--nex", type=int, default=200)
    ap.add_argument("--degree", type=int, default=25)
    ap.add_argument("--interval", default="block_top")
    ap.add_argument("--problems", type=int, default=1)
    ap.add_argument("--generalized", action="store_true")
    ap.add_argument("--max-it", type=int, default=20000)
    ap.add_argument("--out", default="gpurun_out/c4.json")
    ap.add_argument("--ranks", type=int, default=1,
                    help="column-shard every solve over this many in-process ranks "
                         "(devices=[0] * ranks: rank threads sharing cuda:0 -- a check of "
                         "the N-rank code path at full size, not a timing)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    eng = D.Engine.get(dev)
    n = args.n
    t0 = time.perf_counter()
    a, lam = Wl.spectrum_matrix_torch(0, n, dev)
    s = None
    if args.generalized:
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        b = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
        s = torch.empty_like(b)
        eng.zgemm("C", "N", n, n, n, 1.0, b, b, 0.0, s)
        del b
        eng.hermitize(s)
        s.mul_(0.1 / lanczos_norm(eng, s, 2))
        s.diagonal().add_(1.0)
    delta = 1e-3 * max(abs(lam[0]), abs(lam[-1]))
    t_gen = time.perf_counter() - t0
    cfg = G.SolverConfig(nev=args.nev, buffer=args.nex, degree=args.degree,
                         max_outer_iters=args.max_it, interval=args.interval)
    results = {"n": n, "nev": args.nev, "nex": args.nex, "degree": args.degree,
               "interval": args.interval, "generalized": args.generalized, "t_generate_s": t_gen,
               "ranks": args.ranks, "problems": []}
    shard = {"devices": [0] * args.ranks} if args.ranks > 1 else {}
    prev, prior, running = None, None, None
    smat = G.HermitianDenseMatrix.from_device(s, trusted=True) if s is not None else None
    gE = torch.Generator(device=dev)
    for ell in range(1, args.problems + 1):
        if ell > 1:  # A_{ell} = A_{ell-1} + delta E, E Hermitian Gaussian with ||E||_2 ~ 1
            gE.manual_seed(100 + ell)
            e = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=gE)
            e = (e + e.conj().T) / 2
            e = e.conj().resolve_conj().contiguous()
            e.mul_(delta / lanczos_norm(eng, e, 200 + ell))
            a.add_(e)
            del e
            torch.cuda.empty_cache()
        amat = G.HermitianDenseMatrix.from_device(a.clone() if smat is not None else a, trusted=True)
        y0 = None
        solver_rng = np.random.default_rng([0, 11, ell])
        if prev is not None:
            pad_rng = np.random.default_rng([0, 13, ell])
            extra = args.nev + args.nex - prev.s
            pad = pad_rng.standard_normal((n, extra)) + 1j * pad_rng.standard_normal((n, extra))
            y0 = G.VectorBlock(torch.cat([prev.device_block(), D.to_device(pad, dev)], dim=0))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        progress = open(args.out + f".p{ell}.progress", "w")

        def log(it, t1=t1, progress=progress):
            # streamed so a run cut by the call limit still reports how far it got
            if it.iteration % 25 == 0 or it.iteration < 5:
                progress.write(json.dumps({"it": it.iteration, "cols": it.filtered_cols,
                                           "locked": it.converged, "max_res": it.max_resid,
                                           "t": time.perf_counter() - t1}) + "\n")
                progress.flush()

        try:
            if smat is None:
                lamc, vecs, rep = G.chfsi_solve(amat, y0, cfg, prior=prior, seed=solver_rng,
                                                callback=log, **shard)
            else:
                lamc, vecs, rep = G.solve_generalized(amat, smat, y0, cfg, prior=prior,
                                                      seed=solver_rng, callback=log, **shard)
        except G.NotConverged as exc:
            rep = exc.report
            results["problems"].append({
                "problem": ell, "not_converged": True, "s": time.perf_counter() - t1,
                "outer_iterations": rep.outer_iterations, "locked": len(exc.eigenvalues),
                "t_filter": rep.t_filter, "filter_tflops": rep.filter_tflops})
            print(json.dumps(results["problems"][-1]), flush=True)
            break
        dt = time.perf_counter() - t1
        # verification on the device
        vb = vecs.device_block()
        k = vb.shape[0]
        hv = torch.empty_like(vb)
        eng.zgemm("N", "N", n, k, n, 1.0, a, vb, 0.0, hv)
        if smat is None:
            res = eng.residual_norms(hv, vb, lamc)
            gram = torch.empty((k, k), dtype=vb.dtype, device=dev)
            eng.zgemm("C", "N", k, k, n, 1.0, vb, vb, 0.0, gram)
        else:
            sv = torch.empty_like(vb)
            eng.zgemm("N", "N", n, k, n, 1.0, s, vb, 0.0, sv)
            lt = torch.as_tensor(lamc, device=dev).to(vb.dtype)
            res = torch.linalg.vector_norm(hv - sv * lt[:, None], dim=1).cpu().numpy()
            gram = torch.empty((k, k), dtype=vb.dtype, device=dev)
            eng.zgemm("C", "N", k, k, n, 1.0, vb, sv, 0.0, gram)
        orth = float(torch.linalg.matrix_norm(gram - torch.eye(k, dtype=vb.dtype, device=dev)))
        entry = {"problem": ell, "s_per_solve": dt, "outer_iterations": rep.outer_iterations,
                 "total_matmuls": rep.total_matmuls, "t_filter": rep.t_filter, "t_qr": rep.t_qr,
                 "t_rr": rep.t_rr, "filter_tflops": rep.filter_tflops,
                 "t_lanczos": rep.t_lanczos, "t_resid": rep.t_resid,
                 # per-iteration phase times (the input of scripts/scaling_model.py)
                 "iterations": [[i.filtered_cols, i.converged, i.t_filter, i.t_qr, i.t_rr]
                                for i in rep.iterations],
                 "max_residual": float(np.max(res)), "orthonormality": orth,
                 "lam_first": float(lamc[0]), "lam_last": float(lamc[-1])}
        if ell == 1 and smat is None:
            entry["max_rel_eig_err_vs_exact"] = float(np.max(np.abs(lamc - lam[: args.nev]) /
                                                             np.abs(lam[: args.nev])))
        results["problems"].append(entry)
        print(json.dumps(entry), flush=True)
        prev = vecs
        running = rep.est_lam_next if running is None else min(running, rep.est_lam_next)
        prior = (rep.est_lam1, running)
        del hv
    results["total_s"] = sum(p.get("s_per_solve", p.get("s", 0.0)) for p in results["problems"])
    json.dump(results, open(args.out, "w"), indent=1)
    print(json.dumps({"total_s": results["total_s"]}))


if __name__ == "__main__":
    main()
