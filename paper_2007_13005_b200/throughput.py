"""Smol's end-to-end throughput model (host-side arithmetic, no GPU work).

PAPER.md P:785-796 ("Corrected throughput estimation", Eq. 4): when DNN
execution and input preprocessing are pipelined, a configuration C_i with a
cascade of k DNNs D_{i,1..k} runs at approximately

    T_hat(C_i) ~= min( T_preproc(C_i),  1 / sum_j 1 / (alpha_j^{-1} T_exec(D_{i,j})) )

where alpha_j is the fraction of inputs that reach DNN j (alpha_1 = 1 for the
first model of a cascade).  P:1371-1388 (Sec. 7.2) checks the min() model
against measured pipelined throughput and against two alternatives: "DNN
execution only" and "sum" (stage times add, T = 1 / (1/T_pre + 1/T_exec),
the model for stages that share one device).

All throughputs are in the same unit (images/s).  bench.py --eq4 measures
T_preproc (the fused kernel), T_exec (ResNet-50 on the same GPU) and the
pipelined throughput, and reports each model's prediction and error.
"""
from __future__ import annotations

from typing import Sequence


def dnn_stage(t_exec: Sequence[float], alpha: Sequence[float] | None = None) -> float:
    """Throughput of the DNN cascade: 1 / sum_j alpha_j / T_exec_j (Eq. 4's
    second argument; alpha_j^{-1} T_exec_j is stage j's rate in input units)."""
    t_exec = list(t_exec)
    alpha = [1.0] * len(t_exec) if alpha is None else list(alpha)
    if not t_exec or len(alpha) != len(t_exec):
        raise ValueError("t_exec and alpha must be non-empty and of equal length")
    if any(t <= 0 for t in t_exec) or any(not (0.0 <= a <= 1.0) for a in alpha):
        raise ValueError("throughputs must be > 0 and alpha in [0, 1]")
    s = sum(a / t for a, t in zip(alpha, t_exec))
    return float("inf") if s == 0 else 1.0 / s


def eq4_min(t_preproc: float, t_exec: Sequence[float], alpha: Sequence[float] | None = None) -> float:
    """Eq. 4: min(T_preproc, DNN cascade throughput)."""
    if t_preproc <= 0:
        raise ValueError("t_preproc must be > 0")
    return min(t_preproc, dnn_stage(t_exec, alpha))


def sum_model(t_preproc: float, t_exec: Sequence[float], alpha: Sequence[float] | None = None) -> float:
    """The "sum" heuristic of P:1385-1388: stage times per input add up
    (the right model when both stages share one device's cycles)."""
    if t_preproc <= 0:
        raise ValueError("t_preproc must be > 0")
    return 1.0 / (1.0 / t_preproc + 1.0 / dnn_stage(t_exec, alpha))


def exec_only(t_preproc: float, t_exec: Sequence[float], alpha: Sequence[float] | None = None) -> float:
    """The "DNN execution only" heuristic of P:1385-1388 (ignores preprocessing)."""
    return dnn_stage(t_exec, alpha)


def model_errors(measured: float, t_preproc: float, t_exec: Sequence[float],
                 alpha: Sequence[float] | None = None) -> dict:
    """Each model's prediction and relative error |pred - measured| / measured."""
    out = {}
    for name, f in (("min", eq4_min), ("sum", sum_model), ("exec_only", exec_only)):
        p = f(t_preproc, t_exec, alpha)
        out[name] = {"predicted": p, "rel_error": abs(p - measured) / measured}
    return out
