"""CPU tests of the C-ABI library (no GPU compute): every symbol include/rn.h
declares is exported; the host-side logic (GABRA, costing, partitioning,
parameter layout) is bit-identical to the oracle; error codes."""
import os
import random
import re

import pytest

from oracle import gabra as G
from oracle import net as O
from paper_2104_05035_b200 import rn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "rn.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rn_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = rn.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(rn.EXPORTS)


def test_gabra_bit_exact_vs_oracle():
    """C++ == Python over >= 1000 (instance, seed) pairs incl. heterogeneous capacities."""
    r = random.Random(99)
    pairs = 0
    while pairs < 1000:
        n = r.randint(1, 12)
        m = r.randint(1, 5)
        p = [r.randint(0, 200) for _ in range(n)]
        kind = r.random()
        if kind < 0.5:   # heterogeneous, tight
            d = [r.randint(max(max(p), 1), max(max(p), 1) + sum(p) // m + 30) for _ in range(m)]
        else:            # homogeneous (early stop at UB)
            d = G.default_capacities([max(v, 1) for v in p], m)
        kw = dict(seed=r.randint(0, 2 ** 63), pop_size=r.choice([2, 10, 50]), t_max=r.choice([0, 5, 60]),
                  require_all_used=int(r.random() < 0.2), early_stop_at_ub=int(r.random() < 0.7))
        try:
            ref = G.gabra(p, d, **kw)
        except G.Infeasible:
            with pytest.raises(rn.RnError) as e:
                rn.gabra_place(p, d, **kw)
            assert e.value.status == 3
            continue
        got = rn.gabra_place(p, d, **kw)
        assert got[0] == ref[0] and got[1] == ref[1] and got[2] == ref[2], (p, d, kw)
        pairs += 1


def test_gabra_bottleneck_bit_exact_vs_oracle():
    """objective = 1: C++ == Python over 1000 (instance, seed) pairs."""
    r = random.Random(5)
    pairs = 0
    while pairs < 1000:
        n = r.randint(1, 12)
        m = r.randint(1, 5)
        p = [r.randint(0, 200) for _ in range(n)]
        if r.random() < 0.5:
            d = [r.randint(max(max(p), 1), max(max(p), 1) + sum(p) // m + 30) for _ in range(m)]
        else:
            d = G.default_capacities([max(v, 1) for v in p], m)
        kw = dict(seed=r.randint(0, 2 ** 63), pop_size=r.choice([2, 10, 50]), t_max=r.choice([0, 5, 60]),
                  require_all_used=int(r.random() < 0.2), early_stop_at_ub=int(r.random() < 0.7), objective=1)
        try:
            ref = G.gabra(p, d, **kw)
        except G.Infeasible:
            with pytest.raises(rn.RnError) as e:
                rn.gabra_place(p, d, **kw)
            assert e.value.status == 3
            continue
        got = rn.gabra_place(p, d, **kw)
        assert got[0] == ref[0] and got[1] == ref[1] and got[2] == ref[2], (p, d, kw)
        pairs += 1
    with pytest.raises(rn.RnError) as e:
        rn.gabra_place([1, 2], [4, 4], objective=2)
    assert e.value.status == 1


def test_gabra_worked_example_and_errors():
    assert rn.gabra_place([5, 4, 3], [8, 7]) == ([0, 1, 1], 1.625, [5, 7])
    with pytest.raises(rn.RnError) as e:
        rn.gabra_place([9], [8])
    assert e.value.status == 3
    with pytest.raises(rn.RnError) as e:
        rn.gabra_place([1], [0])
    assert e.value.status == 1


@pytest.mark.parametrize("depth,w,dims", [(0, 8, (16, 16, 16)), (18, 64, (91, 109, 91)), (34, 64, (91, 109, 91)),
                                          (18, 16, (24, 20, 28))])
def test_units_params_match_oracle(depth, w, dims):
    d = rn.net_desc(depth, w, dims)
    ul, pf, pl = rn.net_units(d)
    net = O.Net(depth, w, dims)
    costs = O.unit_costs(net.units)
    assert ul == costs
    f, l = G.partition(costs)
    assert pf == f and pl == l
    t, n, nb = rn.net_params(d)
    assert n == net.n_params
    assert [(a, tuple(b), c) for a, b, c in t] == [(a, tuple(b), c) for a, b, c in net.tensors]
    assert nb == sum(net.bn_channels)
    # max_merge_load variant (r34 -> 13 partitions)
    if depth == 34:
        d2 = rn.net_desc(depth, w, dims, max_merge_load=max(costs))
        assert rn.net_units(d2)[1] == G.partition(costs, max_merge_load=max(costs))[0]


def test_schema_errors():
    with pytest.raises(rn.RnError) as e:
        rn.net_units(rn.net_desc(7, 8, (16, 16, 16)))
    assert e.value.status == 2
    with pytest.raises(rn.RnError) as e:
        rn.net_units(rn.net_desc(0, 12, (16, 16, 16)))
    assert e.value.status == 2


@pytest.mark.parametrize("depth,cap", [(18, False), (34, True)])
def test_slack_placement_policy_bit_exact_and_minimal(depth, cap):
    """Reading G4b: rn_gabra_place_slack == oracle place_with_slack (genes, profit,
    loads, capacities, slack) for the configs[3]/[4] partition chains on 2/4/8
    GPUs and both objectives; every configuration is now placeable; and the slack
    chosen is minimal where brute force can check it: at slack - 0.1 no
    capacity-respecting placement exists (every GPU used)."""
    desc = rn.net_desc(depth, 64, (91, 109, 91))
    units, _, loads = rn.net_units(desc)
    if cap:
        _, _, loads = rn.net_units(rn.net_desc(depth, 64, (91, 109, 91), max_merge_load=max(units)))
    for m in (2, 4, 8):
        for obj in (0, 1):
            kw = dict(seed=7, objective=obj, require_all_used=1, init_attempts=4096)
            got = rn.gabra_place_slack(loads, m, **kw)
            ref = G.place_with_slack(loads, m, **kw)
            assert list(got[0]) == list(ref[0]) and got[1] == ref[1] and list(got[2]) == list(ref[2])
            assert list(got[3]) == list(ref[3]) and got[4] == ref[4]
            assert max(got[2]) <= got[3][0]
            s = got[4]
            if s > 1.1 + 1e-9 and m ** len(loads) <= 10 ** 6:
                d = G.default_capacities(loads, m, round(s - 0.1, 1))
                with pytest.raises(G.Infeasible):
                    G.brute_force(loads, d, require_all_used=True)
