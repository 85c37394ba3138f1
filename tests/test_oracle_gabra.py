"""Pins for the oracle's partitioner and GABRA (CPU only): worked examples
(tests/golden), brute force, closed forms on identical GPUs, published PRNG
reference vectors, and the SPEC acceptance criteria used as property tests."""
import json
import os
import random

import pytest

from oracle import gabra as G
from oracle import net as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_prng_reference_vectors():
    gold = json.load(open(os.path.join(GOLD, "prng.json")))
    _, z = G.splitmix64_next(0)
    assert z == int(gold["splitmix64_seed0_first"], 16)
    r = G.Xoshiro256ss(state=gold["xoshiro_state"])
    assert [r.next() for _ in range(4)] == gold["xoshiro_first4"]
    r = G.Xoshiro256ss(seed=1)
    v = [r.u01() for _ in range(1000)]
    assert all(0.0 <= t < 1.0 for t in v)


def test_profit_fitness_examples():
    # SPEC S:134
    c = G.profit_matrix([6, 4], [12, 8])
    assert c == [[0.5, 0.75], [4 / 12, 0.5]]
    assert G.fitness([0, 1], c) == 1.0
    assert G.profit_matrix([0], [5]) == [[0.0]]


def test_repair_examples():
    g = [0, 0]
    assert G.repair(g, [5, 4], [8, 7]) and G.feasible(g, [5, 4], [8, 7])
    g = [0, 1]
    assert G.repair(g, [5, 4], [8, 7]) and g == [0, 1]                         # no-op
    assert not G.repair([0], [9], [8])


def test_partition_examples():
    assert G.partition([100, 1, 1, 100]) == ([0, 1, 3, 4], [100, 2, 100])
    assert G.partition([10, 10, 10, 10]) == ([0, 1, 2, 3, 4], [10, 10, 10, 10])  # S:70 (>= tie)
    assert G.partition([7]) == ([0, 1], [7])
    tiny = O.unit_costs(O.Net(0, 8, (16, 16, 16)).units)
    assert G.partition(tiny) == ([0, 1, 2, 3, 4], tiny)                        # n = 4 (BASELINE configs[0])
    r18 = O.unit_costs(O.Net(18, 64, (91, 109, 91)).units)
    f, l = G.partition(r18)
    assert len(l) == 8 and l[-1] == 3519969284 and sum(l) == sum(r18)
    r34 = O.unit_costs(O.Net(34, 64, (91, 109, 91)).units)
    f, l = G.partition(r34, max_merge_load=max(r34))
    assert len(l) == 13 and max(l) <= max(r34)
    # coverage + scale invariance
    for k in (3, 1000):
        assert G.partition([c * k for c in r18])[0] == G.partition(r18)[0]


def test_worked_instance_gabra_and_bruteforce():
    gold = json.load(open(os.path.join(GOLD, "gabra_worked.json")))
    p, d = gold["p"], gold["d"]
    bg, bv, bl = G.brute_force(p, d)
    assert bg == gold["genes_0based"] and bv == gold["profit"] and bl == gold["loads"]
    hits = 0
    for seed in range(100):
        g, v, l = G.gabra(p, d, seed=seed)
        assert G.feasible(g, p, d)
        hits += (g == gold["genes_0based"] and v == gold["profit"])
    assert hits >= 95
    assert G.brute_force([1], [2, 4])[0] == [0]                                  # S:208 (1/2 > 1/4)
    with pytest.raises(G.Infeasible):
        G.brute_force([9], [8])
    with pytest.raises(G.Infeasible):
        G.gabra([9], [8])


def test_homogeneous_closed_form_C1():
    """Identical capacities: z(X) = sum p / d for every feasible X (finding 3)."""
    loads = O.unit_costs(O.Net(0, 8, (16, 16, 16)).units)
    d = G.default_capacities(loads, 2)
    assert d == [18599117, 18599117]
    g, v, l = G.gabra(loads, d, seed=7)
    assert v == sum(loads) / d[0] or abs(v - sum(loads) / d[0]) < 1e-15
    assert abs(v - 1.737139886802153) < 1e-15
    assert G.feasible(g, loads, d)
    bg, bv, _ = G.brute_force(loads, d)
    assert bg == [0, 0, 1, 0]


def random_instance(r, max_space=300000):
    """Feasible random instance with n <= 10, m <= 4 (m^n bounded to keep the
    pure-Python brute force fast); capacities are heterogeneous so the GA's
    selection/crossover/mutation/repair paths all run."""
    while True:
        n = r.randint(1, 10)
        m = r.randint(1, 4)
        if m ** n > max_space:
            continue
        p = [r.randint(1, 100) for _ in range(n)]
        d = [r.randint(max(p), max(max(p), sum(p) // m + 60)) for _ in range(m)]
        try:
            G.brute_force(p, d)
        except G.Infeasible:
            continue
        return p, d


def test_gabra_vs_bruteforce_acceptance():
    """GABRA >= 0.95 x optimum on >= 90 of 100 random instances (n<=10, m<=4)."""
    r = random.Random(2024)
    good = 0
    for t in range(100):
        p, d = random_instance(r)
        bg, bv, _ = G.brute_force(p, d)
        try:
            g, v, l = G.gabra(p, d, seed=t)
        except G.Infeasible:          # init (A=64 draws + repair) can miss a tight feasible set
            continue
        assert G.feasible(g, p, d)
        assert v <= bv + 1e-12                                                   # oracle dominance
        assert l == G.gpu_loads(g, p, len(d))
        good += v >= 0.95 * bv
    assert good >= 90


def test_determinism_and_scale_covariance():
    r = random.Random(7)
    for t in range(20):
        p, d = random_instance(r)
        a = G.gabra(p, d, seed=11)
        assert a == G.gabra(p, d, seed=11)
        assert G.brute_force(p, d)[0] == G.brute_force([3 * x for x in p], [3 * x for x in d])[0]


def test_require_all_used():
    p, d = [5, 4, 3], [12, 12]
    g, v, l = G.gabra(p, d, seed=3, require_all_used=1, early_stop_at_ub=0)
    assert len(set(g)) == 2
    bg, bv, _ = G.brute_force(p, d, require_all_used=True)
    assert len(set(bg)) == 2


# ----------------------------------------------------------------------------
# bottleneck objective (objective=1; not in the paper)
# ----------------------------------------------------------------------------

def test_bottleneck_worked_instance_by_hand():
    """p = [5, 4, 3], d = [8, 7]: the feasible placements, enumerated by hand,
    with their bottleneck ratios max_j L_j / d_j: (0,1,1) -> max(5/8, 7/7) = 1;
    (1,0,0) -> max(7/8, 5/7) = 7/8; (0,0,1) -> 9/8 > 1 infeasible; (1,1,0) ->
    L = (3, 9): 9 > 7 infeasible; (0,1,0) -> L = (8, 4): max(1, 4/7) = 1;
    (1,0,1) -> L = (4, 8): 8 > 7 infeasible.  Bound lb = max(12/15, 5/8) = 0.8.
    Optimum (1,0,0) with f = 0.8 / (7/8) = 32/35."""
    lb = G.bottleneck_bound([5, 4, 3], [8, 7])
    assert lb == 0.8
    assert G.bottleneck_fitness([0, 1, 1], [5, 4, 3], [8, 7], lb) == 0.8
    assert G.bottleneck_fitness([1, 0, 0], [5, 4, 3], [8, 7], lb) == 0.8 / (7 / 8)
    g, v, loads = G.brute_force([5, 4, 3], [8, 7], objective=1)
    assert g == [1, 0, 0] and loads == [7, 5] and abs(v - 32 / 35) < 1e-15
    g2, v2, _ = G.gabra([5, 4, 3], [8, 7], objective=1)
    assert g2 == [1, 0, 0] and v2 == v


def test_bottleneck_identical_gpus_closed_forms():
    """Identical GPUs: n = m equal partitions -> one per GPU, f = 1 (the bound
    sum p / sum d is met); the tiny network's 4 units on 2 GPUs (configs[0]):
    the bound max p / d is met by isolating the attention module
    (983040 + 14385152 + 32788 = 15400980 <= 16908288), f = 1.  Eq. 3's profit
    is the same for every feasible placement there (finding 3)."""
    p = [100] * 4
    d = G.default_capacities(p, 4)
    g, v, loads = G.gabra(p, d, objective=1)
    assert v == 1.0 and sorted(g) == [0, 1, 2, 3] and loads == [100] * 4
    p = [983040, 14385152, 16908288, 32788]
    d = [18599117, 18599117]
    g, v, loads = G.gabra(p, d, objective=1)
    assert v == 1.0 and sorted(loads) == [15400980, 16908288]
    assert g[2] != g[0] and g[0] == g[1] == g[3]


def test_bottleneck_gabra_vs_bruteforce():
    """The GA under the bottleneck objective: feasible, never above the brute-force
    optimum, and >= 0.95 x optimum on >= 90 of 100 random heterogeneous instances."""
    r = random.Random(77)
    good = total = 0
    for t in range(100):
        p, d = random_instance(r)
        try:
            bg, bv, _ = G.brute_force(p, d, objective=1)
            g, v, l = G.gabra(p, d, seed=t, objective=1)
        except G.Infeasible:
            continue
        total += 1
        assert G.feasible(g, p, d)
        assert v <= bv + 1e-12
        good += v >= 0.95 * bv
    assert total >= 90 and good >= 0.9 * total


def test_init_fallback_worst_fit_decreasing():
    """Reading G19b: with a single random draw per chromosome (init_attempts=1) on
    identical GPUs that only admit permutations (p = [5, 4, 3, 2], d = 5 each,
    require_all_used), the chromosomes that neither the draw nor the repair makes
    feasible are the worst-fit-decreasing one, derived by hand: 5 -> GPU 0 (all
    have 5 free, lowest index), 4 -> GPU 1, 3 -> GPU 2, 2 -> GPU 3."""
    p, d = [5, 4, 3, 2], [5, 5, 5, 5]
    assert G.wfd_chromosome(p, d) == [0, 1, 2, 3]
    # heterogeneous, by hand: 3 (i=0) -> GPU 1 (6 free); 3 (i=1) -> GPU 0 (4 free); 2 -> GPU 1 (3 free)
    assert G.wfd_chromosome([3, 3, 2], [4, 6]) == [1, 0, 1]
    g, v, loads = G.gabra(p, d, require_all_used=1, init_attempts=1, seed=3, early_stop_at_ub=0, t_max=3)
    assert sorted(g) == [0, 1, 2, 3] and sorted(loads) == [2, 3, 4, 5]
    # a capacity that no placement satisfies is still reported infeasible
    with pytest.raises(G.Infeasible):
        G.gabra([6, 1], [5, 5], init_attempts=2)
