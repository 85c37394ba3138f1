"""ORACLE — test infrastructure only (tests/ and tools/ only; the product never
imports it).  Step-time model of the hybrid schedule and the contiguous split
(placement quality on real hardware).

The paper reports measured times (Table 2) and gives the speed-up of
data-parallel training (Eq. 12); SPEC S:255-295 states an
alpha-beta model of a step.  Written out plainly (reading F2 in DESIGN.md):

  stage compute   C_s = sum_{i: genes_i = s} t_i        (t_i: partition i's forward +
                                                          backward per micro-batch,
                                                          measured on the B200)
  boundary p2p    every cut i|i+1 whose partitions sit on different stages moves the
                  activation forward and its gradient back:
                  2 (alpha + b_i / beta) per micro-batch, charged to both stages
  per stage       T_s = C_s + P_s
  pipeline        synchronous (GPipe, M_b micro-batches):  (M_b + S - 1) max_s T_s
                  delayed gradients (f1, all stages busy):  M_b max_s T_s
  all-reduce      ring over the R replicas of a stage (Fig. 3):
                  A_s = 2 (R-1) (g_s / R) / beta + 2 (R-1) alpha,  A = max_s A_s
  step            pipeline + A,  or max(pipeline, A) when the all-reduce overlaps
"""
from __future__ import annotations


def ring_allreduce_time(nbytes: float, m: int, alpha: float, beta: float) -> float:
    """0 for m = 1, else 2(m-1)(nbytes/m)/beta + 2(m-1) alpha."""
    if m <= 1:
        return 0.0
    return 2.0 * (m - 1) * (nbytes / m) / beta + 2.0 * (m - 1) * alpha


def step_time(part_time, cut_bytes, param_bytes, genes, S, R, Mb, alpha, beta, schedule=0, overlap=False):
    """Returns (step, pipeline, allreduce, per-stage T_s).  schedule 0: synchronous
    pipeline (bubble (S-1)/(M_b+S-1)); 1: delayed-gradient pipeline (f1)."""
    n = len(part_time)
    C = [0.0] * S
    Pp = [0.0] * S
    G = [0.0] * S
    for i in range(n):
        C[genes[i]] += part_time[i]
        G[genes[i]] += param_bytes[i]
    for i in range(n - 1):
        if genes[i] != genes[i + 1]:
            c = 2.0 * (alpha + cut_bytes[i] / beta)
            Pp[genes[i]] += c
            Pp[genes[i + 1]] += c
    T = [C[s] + Pp[s] for s in range(S)]
    tmax = max(T)
    pipe = (Mb + S - 1) * tmax if schedule == 0 else Mb * tmax
    A = max(ring_allreduce_time(G[s], R, alpha, beta) for s in range(S))
    step = max(pipe, A) if overlap else pipe + A
    return step, pipe, A, T


def speedup_eq12(T1, Tm, TS1, TSm, E1, Em):
    """Eq. 12 as printed: ST_m = (T_1/T_m) (TS_1/TS_m) (E_1/E_m)."""
    return (T1 / Tm) * (TS1 / TSm) * (E1 / Em)


def contiguous_split(loads, S):
    """Contiguous stages (partitions i..j on one stage, stages in chain order, every
    stage non-empty) minimising the largest stage load: dynamic programme over
    (stages, prefix); among optimal splits the last stage is the shortest possible
    (the largest last cut), recursively.  Returns (genes, max load)."""
    n = len(loads)
    if S < 1 or n < S:
        raise ValueError("need 1 <= S <= n")
    pre = [0]
    for v in loads:
        pre.append(pre[-1] + v)
    INF = float("inf")
    best = [[INF] * (n + 1) for _ in range(S + 1)]
    best[0][0] = 0
    for s in range(1, S + 1):
        for i in range(s, n + 1):
            for j in range(s - 1, i):
                if best[s - 1][j] == INF:
                    continue
                v = max(best[s - 1][j], pre[i] - pre[j])
                if v < best[s][i]:
                    best[s][i] = v
    genes = [0] * n
    i = n
    for s in range(S, 0, -1):
        for j in range(i - 1, s - 2, -1):   # largest j first: shortest last stage
            if best[s - 1][j] != INF and max(best[s - 1][j], pre[i] - pre[j]) == best[s][i]:
                for k in range(j, i):
                    genes[k] = s - 1
                i = j
                break
    return genes, best[S][n]
