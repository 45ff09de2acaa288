"""Table-1-style scaling report (Table 1).

The paper reports, per GPU count, the execution time of one training epoch, the speedup
with respect to the previous row, and the "% scaling w.r.t. 1 GPU".  From the
printed epoch times (6439.93 s on 1 GPU, 3268.65 on 2, ...) those columns are

    speedup_N  = t_prev / t_N                      (1.97x, 1.93x, 2.01x, 1.83x)
    scaling_N  = 100 * t_1 / (N * t_N)             (98.5, 95.0, 95.4, 87.3)

i.e. an epoch over a fixed dataset (strong scaling of the epoch).  A synthetic DP-SGD step
with a fixed per-GPU batch (weak scaling, scripts/train_ddp.py) maps onto the same columns
through the epoch it implies: an epoch of D samples takes D / (N * b) steps, so
t_epoch(N) = t_step(N) * D / (N * b) and scaling_N = 100 * t_step(1) / t_step(N).
Host-side arithmetic only; no GPU.
"""
from __future__ import annotations


def epoch_seconds(step_ms: float, n_gpus: int, batch_per_gpu: int, dataset: int) -> float:
    """Epoch time implied by a weak-scaling step time: D / (N b) steps of step_ms each."""
    return step_ms * 1e-3 * dataset / (n_gpus * batch_per_gpu)


def table1_rows(epoch_times: dict[int, float]) -> list[dict]:
    """Rows of Table 1 from {n_gpus: epoch seconds}, in ascending GPU count: speedup with
    respect to the previous row and % scaling with respect to 1 GPU."""
    ns = sorted(epoch_times)
    if not ns or ns[0] != 1:
        raise ValueError("Table 1 needs the 1-GPU row")
    t1 = epoch_times[1]
    rows, prev = [], None
    for n in ns:
        t = epoch_times[n]
        rows.append({"gpus": n, "seconds": t,
                     "speedup_prev": None if prev is None else epoch_times[prev] / t,
                     "scaling_pct": None if n == 1 else 100.0 * t1 / (n * t)})
        prev = n
    return rows


def format_rows(rows: list[dict], title: str = "") -> str:
    out = [title] if title else []
    out.append(f"{'# GPUs':>6} | {'Execution time (s)':>18} | {'Speedup w.r.t. previous':>23} | "
               f"{'% Scaling w.r.t. 1 GPU':>22}")
    for r in rows:
        sp = "" if r["speedup_prev"] is None else f"{r['speedup_prev']:.2f}x"
        sc = "" if r["scaling_pct"] is None else f"{r['scaling_pct']:.1f}"
        out.append(f"{r['gpus']:>6} | {r['seconds']:>18.2f} | {sp:>23} | {sc:>22}")
    return "\n".join(out)
