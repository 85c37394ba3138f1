// gabra.cpp — Genetic Algorithm Based Resource Allocation (§3.1.2,
// P:170-277): 0-1 multiple knapsack Eqs. 3-8, Algorithm 1 (steady-state GA),
// Algorithm 2 (initial population), fitness, roulette selection
// (P:263), midpoint crossover Algorithm 3, inversion mutation
// (P:277), replace-worst and incumbent update.  Every silent or
// garbled detail follows the pinned text in DESIGN.md "GABRA" (readings
// G1-G23).  Host code only; compiled with -ffp-contract=off so every double
// operation rounds exactly like the oracle's Python floats.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/rn.h"
#include "error.h"

namespace rn {
namespace {

// xoshiro256** seeded by four splitmix64 outputs (reading G20).
struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) {
      st += 0x9E3779B97F4A7C15ull;
      uint64_t z = st;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      s[i] = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  int randint(int k) { return (int)(next() % (uint64_t)k); }
  double u01() { return (double)(next() >> 11) * 0x1.0p-53; }
  bool bern(double q) { return u01() < q; }
};

struct Problem {
  int n, m;
  const int64_t *p;
  const int64_t *d;
  bool U;
  std::vector<double> c;  // c[i*m + j] = p_i / d_j  (Eq. 3, reading G5)

  int objective = 0;  // 0: Eq. 3 profit (the paper); 1: bottleneck
  double lb = 0.0;    // objective 1: max(sum p / sum d, max p / max d)

  double fit(const std::vector<int> &g) const {
    if (objective == 1) {
      // f2: lb / max_j (L_j / d_j) in (0, 1]; max over j ascending, strict >; 1 when all loads are 0
      std::vector<int64_t> L;
      loads(g, L);
      double mr = 0.0;
      for (int j = 0; j < m; ++j) {
        const double r = (double)L[j] / (double)d[j];
        if (r > mr) mr = r;
      }
      return mr == 0.0 ? 1.0 : lb / mr;
    }
    double f = 0.0;  // fitness, left-to-right (G9)
    for (int i = 0; i < n; ++i) f = f + c[(size_t)i * m + g[i]];
    return f;
  }
  void loads(const std::vector<int> &g, std::vector<int64_t> &L) const {
    L.assign(m, 0);
    for (int i = 0; i < n; ++i) L[g[i]] += p[i];
  }
  bool feasible(const std::vector<int> &g) const {  // Eq. 6 (+ P:171 when U)
    std::vector<int64_t> L;
    loads(g, L);
    for (int j = 0; j < m; ++j)
      if (L[j] > d[j]) return false;
    if (U) {
      std::vector<char> used(m, 0);
      for (int i = 0; i < n; ++i) used[g[i]] = 1;
      for (int j = 0; j < m; ++j)
        if (!used[j]) return false;
    }
    return true;
  }
  // Deterministic greedy repair (G14): move the heaviest partition of the
  // lowest-index overloaded GPU to the GPU with most slack, if it fits.
  bool repair(std::vector<int> &g) const {
    std::vector<int64_t> L;
    for (;;) {
      loads(g, L);
      int j = -1;
      for (int k = 0; k < m; ++k)
        if (L[k] > d[k]) { j = k; break; }
      if (j < 0) return feasible(g);
      // members of j sorted by (p desc, i asc): selection scan, stable
      std::vector<int> mem;
      for (int i = 0; i < n; ++i)
        if (g[i] == j) mem.push_back(i);
      for (size_t a = 1; a < mem.size(); ++a) {  // insertion sort, stable
        int v = mem[a];
        size_t b = a;
        while (b > 0 && p[mem[b - 1]] < p[v]) { mem[b] = mem[b - 1]; --b; }
        mem[b] = v;
      }
      bool moved = false;
      for (int i : mem) {
        int best_k = -1;
        int64_t best_slack = 0;
        for (int k = 0; k < m; ++k) {
          if (k == j) continue;
          int64_t sl = d[k] - L[k];
          if (best_k < 0 || sl > best_slack) { best_k = k; best_slack = sl; }
        }
        if (best_k >= 0 && p[i] <= best_slack) {
          g[i] = best_k;
          moved = true;
          break;
        }
      }
      if (!moved) return false;
    }
  }
};

}  // namespace

rn_status gabra_place(int32_t n, const int64_t *loads, int32_t m, const int64_t *caps,
                      const rn_ga_params &gp, int32_t *genes_out, double *profit_out,
                      int64_t *gpu_load_out) {
  Problem pr;
  pr.n = n;
  pr.m = m;
  pr.p = loads;
  pr.d = caps;
  pr.U = gp.require_all_used != 0;
  pr.objective = gp.objective;
  {
    int64_t sp = 0, sd = 0, mp = loads[0], md = caps[0];
    for (int i = 0; i < n; ++i) {
      sp += loads[i];
      if (loads[i] > mp) mp = loads[i];
    }
    for (int j = 0; j < m; ++j) {
      sd += caps[j];
      if (caps[j] > md) md = caps[j];
    }
    const double a = (double)sp / (double)sd, b = (double)mp / (double)md;
    pr.lb = a > b ? a : b;
  }
  pr.c.resize((size_t)n * m);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) pr.c[(size_t)i * m + j] = (double)loads[i] / (double)caps[j];

  const int P = gp.pop_size, T = gp.t_max, R = gp.dup_retries, A = gp.init_attempts;
  const bool E = gp.early_stop_at_ub != 0;
  Rng rng(gp.seed);

  // Algorithm 2: random capacity-respecting chromosomes (G19)
  std::vector<std::vector<int>> pop(P, std::vector<int>(n));
  for (int q = 0; q < P; ++q) {
    bool ok = false;
    std::vector<int> g(n);
    for (int a = 0; a < A && !ok; ++a) {
      for (int i = 0; i < n; ++i) g[i] = rng.randint(m);
      if (pr.feasible(g) || pr.repair(g)) ok = true;
    }
    if (!ok) {
      // reading G19b: A random draws + repair found nothing (tight capacities, or
      // require_all_used with n close to m) -> the deterministic worst-fit-decreasing
      // chromosome (partitions by (p desc, i asc), each to the GPU with the most
      // remaining capacity, lowest index on ties); consumes no random numbers
      std::vector<int> order(n);
      for (int i = 0; i < n; ++i) order[i] = i;
      for (int a = 1; a < n; ++a)  // insertion sort: stable, (p desc, i asc)
        for (int b = a; b > 0 && loads[order[b]] > loads[order[b - 1]]; --b) std::swap(order[b], order[b - 1]);
      std::vector<int64_t> rem(caps, caps + m);
      for (int a = 0; a < n; ++a) {
        int k = 0;
        for (int j = 1; j < m; ++j)
          if (rem[j] > rem[k]) k = j;
        g[order[a]] = k;
        rem[k] -= loads[order[a]];
      }
      ok = pr.feasible(g);
    }
    if (!ok) return set_error(RN_ERR_INFEASIBLE, "GABRA: no capacity-respecting placement found");
    pop[q] = g;
  }
  std::vector<double> f(P);
  for (int q = 0; q < P; ++q) f[q] = pr.fit(pop[q]);
  int bq = 0;
  for (int q = 1; q < P; ++q)
    if (f[q] > f[bq]) bq = q;
  std::vector<int> best = pop[bq];
  double best_val = f[bq];
  double ub = 0.0;
  for (int i = 0; i < n; ++i) {
    double mx = pr.c[(size_t)i * m];
    for (int j = 1; j < m; ++j)
      if (pr.c[(size_t)i * m + j] > mx) mx = pr.c[(size_t)i * m + j];
    ub = ub + mx;
  }
  if (pr.objective == 1) ub = 1.0;  // the bottleneck bound is met

  auto roulette = [&]() -> const std::vector<int> & {
    double tot = 0.0;
    for (int q = 0; q < P; ++q) tot = tot + f[q];
    if (tot <= 0.0) return pop[rng.randint(P)];
    double x = rng.u01() * tot;
    double acc = 0.0;
    for (int q = 0; q < P; ++q) {
      acc = acc + f[q];
      if (x < acc) return pop[q];
    }
    return pop[P - 1];
  };

  if (!(E && best_val == ub)) {
    std::vector<int> W(n);
    for (int t = 0; t < T; ++t) {
      for (int r = 0; r < R; ++r) {
        const std::vector<int> Y1 = roulette();
        const std::vector<int> Y2 = roulette();
        if (rng.bern(gp.p_cross)) {  // Algorithm 3, cp = floor(n/2) (G10)
          const int cp = n / 2;
          for (int i = 0; i < n; ++i) W[i] = i < cp ? Y1[i] : Y2[i];
        } else {
          W = Y1;  // G11
        }
        if (rng.bern(gp.p_mut)) {  // inversion mutation (G12)
          int a = rng.randint(n), b = rng.randint(n);
          if (a > b) { int tmp = a; a = b; b = tmp; }
          while (a < b) { int tmp = W[a]; W[a] = W[b]; W[b] = tmp; ++a; --b; }
        }
        if (!pr.feasible(W) && !pr.repair(W)) continue;
        bool dup = false;
        for (int q = 0; q < P && !dup; ++q) dup = (pop[q] == W);
        if (dup) continue;  // "ignore W and go to" (bounded, G15)
        const double fw = pr.fit(W);
        int z = 0;
        for (int q = 1; q < P; ++q)
          if (f[q] < f[z]) z = q;  // first minimal (G16)
        pop[z] = W;
        f[z] = fw;
        if (fw > best_val) { best = W; best_val = fw; }  // strict (G17)
        break;
      }
      if (E && best_val == ub) break;
    }
  }
  std::vector<int64_t> L;
  pr.loads(best, L);
  for (int i = 0; i < n; ++i) genes_out[i] = best[i];
  if (profit_out) *profit_out = best_val;
  if (gpu_load_out)
    for (int j = 0; j < m; ++j) gpu_load_out[j] = L[j];
  return RN_OK;
}

}  // namespace rn
