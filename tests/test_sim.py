"""f2: the step-time model and the contiguous split — oracle pins
(SPEC S:255-295 examples, Eq. 12 with the paper's Table 2 times, brute force) and
the C-ABI implementation bit-identical to the oracle.  CPU only."""
import itertools
import random

import pytest

from oracle import sim as M
from paper_2104_05035_b200 import rn


def test_ring_allreduce_spec_examples():
    assert M.ring_allreduce_time(1e9, 1, 1e-5, 1e11) == 0.0                    # S:265 m = 1
    assert M.ring_allreduce_time(1000.0, 4, 0.0, 1.0) == 1500.0                # S:266 2*3*(P/4)
    a = M.ring_allreduce_time(1e9, 8, 0.0, 1e11)
    assert abs(M.ring_allreduce_time(1e9, 8, 0.0, 2e11) - a / 2) < 1e-15      # S:267 linear in 1/beta
    assert M.ring_allreduce_time(7.0, 2, 0.0, 1.0) == 7.0                      # S:294 P/B at m = 2


def test_step_time_spec_examples():
    # one device, one partition: L/d, no all-reduce
    st, pipe, ar, T = M.step_time([3.0], [], [100.0], [0], 1, 1, 1, 0.0, 1.0)
    assert (st, pipe, ar) == (3.0, 3.0, 0.0)
    # two equal stages, zero comms: half the single-device time with delayed
    # gradients; the synchronous pipeline with one micro-batch gains nothing
    st1, _, _, _ = M.step_time([1.0, 1.0], [0.0], [0.0, 0.0], [0, 1], 2, 1, 1, 0.0, 1.0, schedule=1)
    st0, _, _, _ = M.step_time([1.0, 1.0], [0.0], [0.0, 0.0], [0, 1], 2, 1, 1, 0.0, 1.0, schedule=0)
    assert st1 == 1.0 and st0 == 2.0
    # bubble (S-1)/(Mb+S-1) of the synchronous schedule
    _, pipe, _, _ = M.step_time([1.0] * 4, [0.0] * 3, [0.0] * 4, [0, 1, 2, 3], 4, 1, 4, 0.0, 1.0)
    assert pipe == 7.0
    # monotone in bandwidth (S invariant)
    prev = None
    for beta in (1e9, 1e10, 1e11):
        st, _, _, _ = M.step_time([1e-3, 2e-3], [1e6], [4e6, 4e6], [0, 1], 2, 4, 2, 1e-5, beta)
        assert prev is None or st <= prev
        prev = st
    # overlap: max instead of sum
    st, pipe, ar, _ = M.step_time([1e-3], [], [1e9], [0], 1, 8, 1, 0.0, 1e11, overlap=True)
    assert st == max(pipe, ar)


def test_eq12_table2():
    # the paper's Table 2 times: ResAttNet34 68 -> 12 min, ResAttNet18 34 -> 6 min
    assert abs(M.speedup_eq12(68, 12, 1, 1, 1, 1) - 68 / 12) < 1e-12
    assert abs(M.speedup_eq12(34, 6, 1, 1, 1, 1) - 34 / 6) < 1e-12
    # m identical devices, balanced, zero comms: data-parallel speed-up m:
    # same step time, m x fewer steps per epoch
    m = 8
    t1, _, _, _ = M.step_time([1.0], [], [1.0], [0], 1, 1, 1, 0.0, 1.0)
    tm, _, _, _ = M.step_time([1.0], [], [1.0], [0], 1, m, 1, 0.0, float("inf"))
    assert M.speedup_eq12(t1, tm, 120 / 6, 120 / (6 * m), 1, 1) == m


def test_contiguous_split_vs_brute_force():
    r = random.Random(5)
    for _ in range(200):
        n = r.randint(1, 9)
        S = r.randint(1, n)
        loads = [r.randint(0, 50) for _ in range(n)]
        genes, mx = M.contiguous_split(loads, S)
        assert all(genes[i] <= genes[i + 1] for i in range(n - 1)) and sorted(set(genes)) == list(range(S))
        assert max(sum(loads[i] for i in range(n) if genes[i] == s) for s in range(S)) == mx
        best = min(max(sum(loads[a:b]) for a, b in zip((0,) + cuts, cuts + (n,)))
                   for cuts in itertools.combinations(range(1, n), S - 1))
        assert mx == best
        g2, mx2 = rn.contiguous_split(loads, S)
        assert g2 == genes and mx2 == mx


def test_simulator_bit_identical_to_oracle():
    r = random.Random(9)
    for _ in range(300):
        n = r.randint(1, 13)
        S = r.randint(1, min(n, 8))
        genes = [r.randrange(S) for _ in range(n)]
        pt = [r.uniform(1e-5, 1e-3) for _ in range(n)]
        cb = [r.uniform(0, 2e7) for _ in range(n - 1)]
        pb = [r.uniform(0, 2e8) for _ in range(n)]
        R, Mb = r.randint(1, 8), r.randint(1, 4)
        kw = dict(schedule=r.randint(0, 1), overlap=bool(r.randint(0, 1)))
        a = M.step_time(pt, cb, pb, genes, S, R, Mb, 5e-6, 4.5e11, **kw)
        b = rn.simulate_step(pt, cb, pb, genes, S, R, Mb, 5e-6, 4.5e11, **kw)
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2] and list(a[3]) == b[3]


def test_simulator_rejects_bad_input():
    with pytest.raises(rn.RnError):
        rn.simulate_step([1.0], [], [1.0], [1], 1, 1, 1, 0.0, 1.0)        # gene out of range
    with pytest.raises(rn.RnError):
        rn.contiguous_split([1, 2], 3)                                    # n < S
