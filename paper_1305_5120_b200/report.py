"""CSV surfaces of a solve, with the reference's column schemas so GPU runs can be
diffed against CPU runs: per-iteration report (cli.py:32-35, :89-103), sequence
table (cli.py:36-38, :169-211) and phase breakdown (bench.py:30, :57-82).
"""

__all__ = ["REPORT_HEADER", "SEQUENCE_HEADER", "PHASES_HEADER", "report_csv_text",
           "sequence_csv_text", "phase_rows", "rows_to_csv"]

REPORT_HEADER = ["iter", "filtered_cols", "converged", "max_resid", "matmul_count",
                 "t_filter", "t_qr", "t_rr", "t_resid"]
SEQUENCE_HEADER = ["cycle", "work_random", "work_reuse", "work_ratio", "median_angle"]
PHASES_HEADER = ["phase", "seconds", "fraction", "config_hash"]


def rows_to_csv(header, rows):
    return "\n".join([",".join(header)] + [",".join(str(x) for x in r) for r in rows]) + "\n"


def report_csv_text(report):
    """One row per outer iteration; the first five columns are deterministic
    (reference criterion 7 compares exactly those across repeated runs)."""
    rows = [(it.iteration, it.filtered_cols, it.converged, f"{it.max_resid:.6e}", it.matmuls,
             f"{it.t_filter:.6f}", f"{it.t_qr:.6f}", f"{it.t_rr:.6f}", f"{it.t_resid:.6f}")
            for it in report.iterations]
    return rows_to_csv(REPORT_HEADER, rows)


def _opt(x, fmt):
    return format(x, fmt) if x is not None else ""


def sequence_csv_text(random_report=None, reuse_report=None, ratios=None):
    """Per-cycle work (random / reuse), work ratio and median reuse angle."""
    base = reuse_report if reuse_report is not None else random_report
    if base is None:
        return rows_to_csv(SEQUENCE_HEADER, [])
    ncyc = len(base.work)
    ratios = ratios if ratios is not None else [None] * ncyc
    med = base.median_angles()
    rows = []
    for i in range(ncyc):
        wr = random_report.work[i] if random_report is not None else None
        wu = reuse_report.work[i] if reuse_report is not None else None
        rows.append((i + 1, "" if wr is None else wr, "" if wu is None else wu,
                     _opt(ratios[i], ".4f"), _opt(med[i], ".6e")))
    return rows_to_csv(SEQUENCE_HEADER, rows)


def phase_rows(report, total_seconds, config_hash=""):
    """(phase, seconds, fraction, hash) rows like bench_phases: filter, qr,
    rayleigh_ritz, residuals and "other" (Lanczos, locking, allocation)."""
    named = {"filter": report.t_filter, "qr": report.t_qr, "rayleigh_ritz": report.t_rr,
             "residuals": report.t_resid}
    named["other"] = max(0.0, total_seconds - sum(named.values()))
    return [(ph, f"{s:.6f}", f"{s / total_seconds:.6f}", config_hash) for ph, s in named.items()]
