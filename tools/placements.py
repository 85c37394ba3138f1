"""GABRA placements of the BASELINE hybrid configurations (configs[3], configs[4])
through librn, under the paper's Eq. 3 objective (objective 0) and the bottleneck
objective of SURVEY §8(f) f2 (objective 1): per-GPU loads, bottleneck load
max_j L_j / d_j relative to the bound, and the number of stage hops (cuts in the
partition chain whose two sides sit on different GPUs).  Host only (no GPU).
Usage: python tools/placements.py [seeds=7,8,9,10,11]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_05035_b200 import rn  # noqa: E402

seeds = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "7,8,9,10,11").split(",")]
dims = (91, 109, 91)
cases = [("r18 (configs[3])", 18, 0, [2, 4, 8]), ("r34 (configs[4])", 34, -1, [2, 4, 8])]
for name, depth, cap, ms in cases:
    units, first, loads = rn.net_units(rn.net_desc(depth, 64, dims))
    if cap < 0:  # r34: cap merged light partitions at the heaviest singleton
        units, first, loads = rn.net_units(rn.net_desc(depth, 64, dims, max_merge_load=max(units)))
    print(f"{name}: n = {len(loads)} partitions, loads = {loads}")
    for m in ms:
        for obj in (0, 1):
            for seed in seeds:
                try:  # reading G4b: the smallest slack 1.1, 1.2, ... with a feasible placement
                    g, f, L, d, slack = rn.gabra_place_slack(loads, m, seed=seed, objective=obj,
                                                             require_all_used=1, init_attempts=4096)
                except rn.RnError as e:
                    print(f"  m={m} objective={obj} seed={seed}: {e}")
                    continue
                worst = max(L[j] / d[j] for j in range(m))
                bound = max(sum(loads) / sum(d), max(loads) / max(d))
                hops = sum(1 for i in range(len(g) - 1) if g[i] != g[i + 1])
                print(f"  m={m} objective={obj} seed={seed}: slack={slack:.1f} genes={g} f={f:.6f} loads={L} "
                      f"bottleneck/bound={worst / bound:.4f} hops={hops}")
