"""Kernel-time shares from an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv <command>`), grouped by kernel family.

    python scripts/launch_shares.py X.csv [--skip-torch] > summary.json
"""
import csv
import json
import re
import sys
from collections import defaultdict

UNITS = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "s": 1.0, "second": 1.0}


def family(name):
    if "zgemm_tma_kernel" in name:
        # template args: BM, BN, WM, WN, STAGES, EPI, MINB, MUL, SUMS
        m = re.search(r"zgemm_tma_kernel<([^>]*)>", name)
        args = [a.strip() for a in m.group(1).split(",")] if m else []
        epi = {"0": "store", "1": "filter", "2": "split-K partial"}.get(args[5] if len(args) > 5 else "", "?")
        mul = args[7] if len(args) > 7 else "4"
        sums = len(args) > 8 and args[8] in ("1", "true")
        return f"zgemm_tma {epi} ({'3M' if mul == '3' else '4M'}{', sum planes' if sums else ''})"
    if "zgemm_dmma_kernel" in name:
        return "zgemm_dmma (cp.async, four products)"
    if "splitk_reduce" in name:
        return "split-K reduce"
    if "sum_plane" in name:
        return "sum planes"
    for key in ("residual", "zdotc", "finish_", "hermit", "trtri", "clean_lower", "axpby",
                "mirror", "real_diag", "shift_diag", "sum_pairs", "peak_"):
        if key in name:
            return "chfsi " + key.rstrip("_")
    if any(s in name for s in ("syevd", "heevd", "sytrd", "hetrd", "stedc", "ormtr", "unmtr",
                               "steqr", "potrf", "trsm", "trmm", "geqr", "larf", "lacpy",
                               "laset", "cusolver", "zher", "zgemv", "gemv")):
        return "cuSOLVER / cuBLAS (k x k eigensolve, Cholesky)"
    if "cutlass" in name or "gemm" in name.lower():
        return "library GEMM (torch setup)"
    return "other (torch setup / copies)"


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    t = defaultdict(float)
    c = defaultdict(int)
    for r in rows[1:]:
        f = family(r[ik])
        t[f] += float(r[iv].replace(",", "")) * UNITS[r[iu]]
        c[f] += 1
    if "--skip-torch" in sys.argv:
        for f in [f for f in t if f.startswith(("other", "library"))]:
            del t[f]
    tot = sum(t.values())
    out = {"total_kernel_s": tot, "families": [
        {"family": f, "launches": c[f], "seconds": t[f], "share": t[f] / tot}
        for f in sorted(t, key=t.get, reverse=True)]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
