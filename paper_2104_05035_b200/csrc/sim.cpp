// sim.cpp — step-time model of the hybrid schedule and the contiguous split
// (placement quality on real hardware; SPEC S:255-295 alpha-beta
// model; ring all-reduce P:284 / Fig. 3; Eq. 12).  Host only.  The
// per-partition times it takes are measured on the B200 (rn_query unit_ms_* of a
// timed step), so the model is calibrated on the hardware it plans for.
#include <algorithm>
#include <limits>
#include <vector>

#include "../../include/rn.h"
#include "error.h"
#include "net.h"

namespace rn {

double ring_allreduce_time(double nbytes, int m, double alpha, double beta) {
  if (m <= 1) return 0.0;
  return 2.0 * (m - 1) * (nbytes / m) / beta + 2.0 * (m - 1) * alpha;
}

// same operation order as oracle/sim.py step_time (bit-identical doubles)
void simulate_step(const rn_sim_desc &d, double *step, double *pipe, double *ar, double *stage_t) {
  const int n = d.n, S = d.n_stages;
  std::vector<double> C(S, 0.0), Pp(S, 0.0), G(S, 0.0);
  for (int i = 0; i < n; ++i) {
    C[d.genes[i]] += d.part_time[i];
    G[d.genes[i]] += d.param_bytes[i];
  }
  for (int i = 0; i + 1 < n; ++i)
    if (d.genes[i] != d.genes[i + 1]) {
      const double c = 2.0 * (d.alpha + d.cut_bytes[i] / d.beta);
      Pp[d.genes[i]] += c;
      Pp[d.genes[i + 1]] += c;
    }
  double tmax = -std::numeric_limits<double>::infinity();
  for (int s = 0; s < S; ++s) {
    const double T = C[s] + Pp[s];
    if (stage_t) stage_t[s] = T;
    tmax = std::max(tmax, T);
  }
  const double p = d.schedule == 0 ? (d.micro_batches + S - 1) * tmax : d.micro_batches * tmax;
  double A = -std::numeric_limits<double>::infinity();
  for (int s = 0; s < S; ++s) A = std::max(A, ring_allreduce_time(G[s], d.replicas, d.alpha, d.beta));
  *pipe = p;
  *ar = A;
  *step = d.overlap ? std::max(p, A) : p + A;
}

void contiguous_split(int n, const int64_t *loads, int S, int32_t *genes, int64_t *max_load) {
  std::vector<int64_t> pre(n + 1, 0);
  for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + loads[i];
  const int64_t INF = std::numeric_limits<int64_t>::max();
  std::vector<std::vector<int64_t>> best(S + 1, std::vector<int64_t>(n + 1, INF));
  best[0][0] = 0;
  for (int s = 1; s <= S; ++s)
    for (int i = s; i <= n; ++i)
      for (int j = s - 1; j < i; ++j) {
        if (best[s - 1][j] == INF) continue;
        const int64_t v = std::max(best[s - 1][j], pre[i] - pre[j]);
        if (v < best[s][i]) best[s][i] = v;
      }
  int i = n;
  for (int s = S; s >= 1; --s)
    for (int j = i - 1; j >= s - 1; --j) {  // largest j first: the shortest last stage
      if (best[s - 1][j] != INF && std::max(best[s - 1][j], pre[i] - pre[j]) == best[s][i]) {
        for (int k = j; k < i; ++k) genes[k] = s - 1;
        i = j;
        break;
      }
    }
  if (max_load) *max_load = best[S][n];
}

}  // namespace rn
