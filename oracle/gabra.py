"""ORACLE — test infrastructure only (see oracle/net.py header).

Network partitioning (§3.1.1) and the Genetic
Algorithm Based Resource Allocation GABRA (§3.1.2: Eqs. 3-8,
Algorithms 1-3, the fitness equation, roulette selection P:263, midpoint
crossover P:265-275, inversion mutation P:277) written step by step in the
paper's order, with every silence/garble resolved by the pinned text of
SURVEY §8(c) (readings G1-G23).  Also the exhaustive allocator used
to pin GABRA's optimality (brute force over all m^n assignments).

Pure Python integers/floats; no code shared with the C++ implementation in
paper_2104_05035_b200/csrc/gabra.cpp — both follow the same written text.
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1

RN_OK, RN_ERR_ARG, RN_ERR_SCHEMA, RN_ERR_INFEASIBLE, RN_ERR_NUMERIC = 0, 1, 2, 3, 4
RN_ERR_SIZE = 8


class Infeasible(Exception):
    pass


# ----------------------------------------------------------------------------
# Partitioning ("highly functional layers are partitioned individually",
# P:156 contiguous p_i = {s_i .. s_{i+1}-1}; reading G1: alpha-rule with >=)
# ----------------------------------------------------------------------------

def partition(costs, alpha: float = 1.0, max_merge_load: int = 0):
    """costs: per-unit int loads.  Returns (first_unit list of length n+1, loads).
    A unit with cost >= alpha * mean(costs) is a singleton partition; maximal runs
    of light units merge into one partition, split greedily left to right so a
    merged partition's load never exceeds max_merge_load (0 = no cap) unless a
    single unit alone exceeds it."""
    n = len(costs)
    if n == 0:
        raise ValueError("empty network")
    mean = sum(costs) / n
    heavy = [c >= alpha * mean for c in costs]
    firsts, loads = [], []
    i = 0
    while i < n:
        if heavy[i]:
            firsts.append(i)
            loads.append(costs[i])
            i += 1
            continue
        start, acc = i, 0
        while i < n and not heavy[i]:
            if max_merge_load > 0 and i > start and acc + costs[i] > max_merge_load:
                firsts.append(start)
                loads.append(acc)
                start, acc = i, 0
            acc += costs[i]
            i += 1
        firsts.append(start)
        loads.append(acc)
    firsts.append(n)
    return firsts, loads


def default_capacities(loads, m: int, slack: float = 1.10):
    """Reading G4: d_j = ceil(slack * max(max_i p_i, ceil(sum p / m))) for all j."""
    import math
    tot = sum(loads)
    base = max(max(loads), -(-tot // m))
    return [int(math.ceil(slack * base))] * m


def place_with_slack(loads, m: int, **kw):
    """Reading G4b: the paper gives no capacities for identical GPUs
    (P:171-216).  Take the G4 capacities with the smallest slack s in 1.1, 1.2,
    ..., 2.0 (k/10, k = 11..20) for which Algorithm 1 (with the Algorithm 2
    fallback, G19b) finds a capacity-respecting placement: a partition chain
    whose blocks are too coarse to pack at 10 % slack (r18 on 4 GPUs, r34 on 8)
    is placed at the next slack instead of being declared infeasible.
    Returns (genes, profit, per-GPU loads, capacities, slack)."""
    for k in range(11, 21):
        s = k / 10
        d = default_capacities(loads, m, s)
        try:
            g, f, L = gabra(loads, d, **kw)
        except Infeasible:
            continue
        return g, f, L, d, s
    raise Infeasible("no capacity-respecting placement up to slack 2.0")


# ----------------------------------------------------------------------------
# PRNG (reading G20): xoshiro256** seeded by splitmix64
# ----------------------------------------------------------------------------

def splitmix64_next(state: int):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def _rotl(x, k):
    return ((x << k) | (x >> (64 - k))) & MASK64


class Xoshiro256ss:
    def __init__(self, seed: int | None = None, state=None):
        if state is not None:
            self.s = [int(v) & MASK64 for v in state]
        else:
            st = seed & MASK64
            self.s = []
            for _ in range(4):
                st, z = splitmix64_next(st)
                self.s.append(z)

    def next(self) -> int:
        s = self.s
        result = (_rotl((s[1] * 5) & MASK64, 7) * 9) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def randint(self, k: int) -> int:
        return self.next() % k

    def u01(self) -> float:
        return (self.next() >> 11) * (2.0 ** -53)

    def bern(self, q: float) -> bool:
        return self.u01() < q


# ----------------------------------------------------------------------------
# Knapsack model pieces (Eqs. 3-8)
# ----------------------------------------------------------------------------

def profit_matrix(p, d):
    """Eq. 3: c_ij = p_i / d_j (i = partition, j = GPU; reading G5)."""
    if any(v <= 0 for v in d):
        raise ValueError("capacity must be > 0")
    return [[float(pi) / float(dj) for dj in d] for pi in p]


def profit_fitness(genes, c):
    """Fitness equation (reading G9): f = sum_i c[i][gene_i], left to right."""
    f = 0.0
    for i, g in enumerate(genes):
        f = f + c[i][g]
    return f


fitness = profit_fitness


def bottleneck_bound(p, d):
    """SURVEY §8(f) f2 (not in the paper): lower bound of the bottleneck load
    ratio max_j L_j / d_j over all placements — max(sum p / sum d, max p / max d)
    (the work must fit the total capacity; the largest partition sits somewhere)."""
    sp, sd = 0, 0
    for v in p:
        sp += v
    for v in d:
        sd += v
    a = float(sp) / float(sd)
    b = float(max(p)) / float(max(d))
    return a if a > b else b


def bottleneck_fitness(genes, p, d, lb):
    """f2 objective: f = lb / max_j (L_j / d_j) in (0, 1] (1 = the bound is met);
    the GA maximises it, i.e. minimises the slowest GPU's normalised load — the
    pipeline step time on identical GPUs, where Eq. 3's profit is flat
    (finding 3).  max over j ascending with strict >; f = 1 when every load is 0."""
    m = len(d)
    load = gpu_loads(genes, p, m)
    mr = 0.0
    for j in range(m):
        r = float(load[j]) / float(d[j])
        if r > mr:
            mr = r
    if mr == 0.0:
        return 1.0
    return lb / mr


def gpu_loads(genes, p, m):
    load = [0] * m
    for i, g in enumerate(genes):
        load[g] += p[i]
    return load


def feasible(genes, p, d, require_all_used=False):
    """Eq. 6 capacity (and, with require_all_used, P:171 'each GPU runs at least
    one partition', reading G7).  Eq. 7 holds by the gene encoding."""
    m = len(d)
    load = gpu_loads(genes, p, m)
    if any(load[j] > d[j] for j in range(m)):
        return False
    if require_all_used:
        used = [False] * m
        for g in genes:
            used[g] = True
        if not all(used):
            return False
    return True


def repair(genes, p, d, require_all_used=False):
    """Deterministic greedy repair (reading G14): modifies genes in
    place; returns True iff the result satisfies feasible() in full."""
    m, n = len(d), len(genes)
    while True:
        load = gpu_loads(genes, p, m)
        over = [j for j in range(m) if load[j] > d[j]]
        if not over:
            return feasible(genes, p, d, require_all_used)
        j = over[0]
        members = sorted([i for i in range(n) if genes[i] == j], key=lambda i: (-p[i], i))
        moved = False
        for i in members:
            best_k, best_slack = -1, None
            for k in range(m):
                if k == j:
                    continue
                sl = d[k] - load[k]
                if best_slack is None or sl > best_slack:
                    best_k, best_slack = k, sl
            if best_k >= 0 and p[i] <= best_slack:
                genes[i] = best_k
                moved = True
                break
        if not moved:
            return False


# ----------------------------------------------------------------------------
# GABRA (Algorithm 1), pinned step by step
# ----------------------------------------------------------------------------

def wfd_chromosome(p, d):
    """Reading G19b: worst-fit decreasing — partitions by (p desc, i asc), each to
    the GPU with the most remaining capacity (lowest index on ties)."""
    n, m = len(p), len(d)
    g = [0] * n
    rem = list(d)
    for i in sorted(range(n), key=lambda i: (-p[i], i)):
        k = 0
        for j in range(1, m):
            if rem[j] > rem[k]:
                k = j
        g[i] = k
        rem[k] -= p[i]
    return g


DEFAULT_PARAMS = dict(pop_size=50, t_max=500, p_cross=0.8, p_mut=0.1, seed=7,
                      dup_retries=20, init_attempts=64, require_all_used=0, early_stop_at_ub=1,
                      objective=0)


def gabra(p, d, **kw):
    """Returns (genes 0-based, profit, per-GPU loads).  Raises Infeasible."""
    prm = dict(DEFAULT_PARAMS)
    prm.update(kw)
    P, T = prm["pop_size"], prm["t_max"]
    pc, pm = prm["p_cross"], prm["p_mut"]
    R, A = prm["dup_retries"], prm["init_attempts"]
    U, E = bool(prm["require_all_used"]), bool(prm["early_stop_at_ub"])
    n, m = len(p), len(d)
    if n < 1 or m < 1 or P < 2:
        raise ValueError("bad sizes")
    rng = Xoshiro256ss(prm["seed"])
    c = profit_matrix(p, d)                                   # Algorithm 1 line 1
    obj = int(prm["objective"])
    if obj not in (0, 1):
        raise ValueError("objective must be 0 (Eq. 3) or 1 (bottleneck, SURVEY f2)")
    lb = bottleneck_bound(p, d) if obj == 1 else 0.0

    def fitness(genes, c):                                    # objective 0: Eq. 3 profit
        if obj == 1:
            return bottleneck_fitness(genes, p, d, lb)
        return profit_fitness(genes, c)

    # initial population (Algorithm 2; reading G19)
    pop = []
    for q in range(P):
        accepted = None
        for a in range(A):
            g = [rng.randint(m) for _ in range(n)]
            if feasible(g, p, d, U) or repair(g, p, d, U):
                accepted = g
                break
        if accepted is None:
            # reading G19b: the deterministic worst-fit-decreasing chromosome
            # (partitions by (p desc, i asc), each to the GPU with the most
            # remaining capacity, lowest index on ties); no random numbers
            g = wfd_chromosome(p, d)
            if feasible(g, p, d, U):
                accepted = g
        if accepted is None:
            raise Infeasible("no capacity-respecting placement found")
        pop.append(accepted)
    f = [fitness(g, c) for g in pop]                          # evaluate P(t)
    best_q = 0
    for q in range(1, P):                                     # Z*: first maximal (reading G21)
        if f[q] > f[best_q]:
            best_q = q
    best, best_val = list(pop[best_q]), f[best_q]
    ub = 0.0
    for i in range(n):
        ub = ub + max(c[i])
    if obj == 1:
        ub = 1.0                                              # the bottleneck bound is met
    if E and best_val == ub:                                  # P:277 "optimal profit obtained"
        return best, best_val, gpu_loads(best, p, m)

    def roulette():                                           # phi, P:230 / P:263
        tot = 0.0
        for v in f:
            tot = tot + v
        if tot <= 0.0:
            return pop[rng.randint(P)]
        x = rng.u01() * tot
        acc = 0.0
        for q in range(P):
            acc = acc + f[q]
            if x < acc:
                return pop[q]
        return pop[P - 1]

    for t in range(T):                                        # while t < t_max
        for r in range(R):                                    # bounded "go to" (reading G15)
            Y1 = roulette()
            Y2 = roulette()
            if rng.bern(pc):                                  # Algorithm 3, cp = floor(n/2) (G10)
                cp = n // 2
                W = list(Y1[:cp]) + list(Y2[cp:])
            else:
                W = list(Y1)                                  # reading G11
            if rng.bern(pm):                                  # inversion mutation (G12)
                a = rng.randint(n)
                b = rng.randint(n)
                if a > b:
                    a, b = b, a
                W[a:b + 1] = W[a:b + 1][::-1]
            if not feasible(W, p, d, U) and not repair(W, p, d, U):
                continue
            if any(W == z for z in pop):                      # "ignore W and go to"
                continue
            fw = fitness(W, c)
            z = 0
            for q in range(1, P):                             # Z': first minimal (G16)
                if f[q] < f[z]:
                    z = q
            pop[z] = W
            f[z] = fw
            if fw > best_val:                                 # strict (G17)
                best, best_val = list(W), fw
            break
        if E and best_val == ub:
            break
    return best, best_val, gpu_loads(best, p, m)


def brute_force(p, d, require_all_used=False, limit=10 ** 7, objective=0):
    """Exhaustive Eq. 5 maximiser (objective 0) or bottleneck maximiser
    (objective 1, f2) over all m^n assignments (gene 0 most significant);
    ties -> lexicographically smallest (first found, strict >)."""
    n, m = len(p), len(d)
    if m ** n > limit:
        raise OverflowError("instance too large")
    c = profit_matrix(p, d)
    lb = bottleneck_bound(p, d)

    def fitness(genes, c):
        return bottleneck_fitness(genes, p, d, lb) if objective == 1 else profit_fitness(genes, c)
    best, best_val = None, None
    genes = [0] * n
    for code in range(m ** n):
        x = code
        for i in range(n - 1, -1, -1):
            genes[i] = x % m
            x //= m
        if not feasible(genes, p, d, require_all_used):
            continue
        v = fitness(genes, c)
        if best_val is None or v > best_val:
            best, best_val = list(genes), v
    if best is None:
        raise Infeasible("no feasible assignment")
    return best, best_val, gpu_loads(best, p, m)
