"""Per-iteration trace of the CSC iteration (SURVEY.md §5 "tracing"; the Fig.1 caption reports the time
per iteration and the objective).

One row per iteration of Alg.1:

    iter, F, fit, l1, nnz, tau_z, tau_d, ms_code, ms_filter, ms_obj, ms_iter

F = fit + l1 is the objective (Eq.1) after the iteration's filter step, nnz the number of nonzero codes,
tau_z / tau_d the step sizes the iteration used, and ms_* the device time of each phase, taken with CUDA
events on the context's stream (the same clock bench.py uses).  The phases run as the separate C-ABI
entry points csc_code_step, csc_filter_step and csc_objective -- the same kernels csc_iterate enqueues --
so a traced run computes exactly what an untraced run computes; only the host synchronisations that read
the step sizes and nnz are added (observability, not the benchmarked path).

    from paper_1909_00145_b200.trace import IterationTrace, run_traced
    tr = run_traced(ctx, x, d, z, lam, p, seed, iters=50)
    tr.write_csv("trace.csv")
"""
from __future__ import annotations

import csv
import io
from typing import Dict, Iterable, List, Optional

FIELDS = ("iter", "F", "fit", "l1", "nnz", "tau_z", "tau_d", "ms_code", "ms_filter", "ms_obj", "ms_iter")


class IterationTrace:
    """Rows of the per-iteration trace; CSV with the FIELDS header."""

    def __init__(self) -> None:
        self.rows: List[Dict[str, float]] = []

    def add(self, **row) -> None:
        missing = [f for f in FIELDS if f not in row]
        extra = [f for f in row if f not in FIELDS]
        if missing or extra:
            raise ValueError(f"trace row: missing {missing}, unknown {extra}")
        self.rows.append({f: row[f] for f in FIELDS})

    def __len__(self) -> int:
        return len(self.rows)

    def column(self, name: str) -> List[float]:
        return [r[name] for r in self.rows]

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=FIELDS, lineterminator="\n")
        w.writeheader()
        for r in self.rows:
            w.writerow({k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()})
        return buf.getvalue()

    def write_csv(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.to_csv())

    @staticmethod
    def read_csv(text_or_lines: Iterable[str] | str) -> "IterationTrace":
        lines = text_or_lines.splitlines() if isinstance(text_or_lines, str) else list(text_or_lines)
        rd = csv.DictReader(lines)
        if tuple(rd.fieldnames or ()) != FIELDS:
            raise ValueError(f"trace header {rd.fieldnames} != {FIELDS}")
        tr = IterationTrace()
        for r in rd:
            tr.add(**{k: (int(v) if k in ("iter", "nnz") else float(v)) for k, v in r.items()})
        return tr


def run_traced(ctx, x, d, z, lam: float, p: float, seed: int, iters: int, *, start_iter: int = 0,
               step_z: float = 0.0, step_d: float = 0.0, trace: Optional[IterationTrace] = None,
               on_row=None) -> IterationTrace:
    """Run `iters` iterations (mask iterations start_iter, start_iter + 1, ...) through the C ABI and
    record one trace row per iteration.  on_row(row) is called after each row (e.g. to stream a CSV).
    Between iterations the NCCL communicator is polled for asynchronous errors (csc_comm_check)."""
    import torch
    tr = trace if trace is not None else IterationTrace()
    st = ctx.stream
    for i in range(iters):
        it = start_iter + i
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(st)
        tau_z = ctx.code_step(x, d, z, lam, p, seed, it, step_z=step_z, want_step=True)
        ev[1].record(st)
        tau_d = ctx.filter_step(x, d, z, step_d=step_d, want_step=True)
        ev[2].record(st)
        F, fit, l1 = ctx.objective(x, d, z, lam)
        ev[3].record(st)
        nnz = ctx.count_nonzero(z) if ctx.n_local else 0
        ev[3].synchronize()
        ctx.comm_check()
        row = dict(iter=it, F=F, fit=fit, l1=l1, nnz=nnz, tau_z=tau_z, tau_d=tau_d,
                   ms_code=ev[0].elapsed_time(ev[1]), ms_filter=ev[1].elapsed_time(ev[2]),
                   ms_obj=ev[2].elapsed_time(ev[3]), ms_iter=ev[0].elapsed_time(ev[3]))
        tr.add(**row)
        if on_row is not None:
            on_row(row)
    return tr
