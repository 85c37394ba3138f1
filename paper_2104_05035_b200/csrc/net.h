// net.h — internal (C++) description of 3D-ResAttNet: units, shapes, parameter
// tensors, per-unit costs and partitioning.  Independent re-statement of the
// network described at PAPER.md:364-366 with the readings X1-X11;
// shares no code with oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rn.h"

namespace rn {

struct Dims {
  int d = 1, h = 1, w = 1;
  int64_t vol() const { return (int64_t)d * h * w; }
  bool operator==(const Dims &o) const { return d == o.d && h == o.h && w == o.w; }
};

inline int conv_out(int n, int k, int s, int p) { return (n + 2 * p - k) / s + 1; }
inline Dims conv_out(Dims a, int k, int s, int p) {
  return Dims{conv_out(a.d, k, s, p), conv_out(a.h, k, s, p), conv_out(a.w, k, s, p)};
}

enum UnitKind { U_STEM = 0, U_BLOCK = 1, U_ATT = 2, U_HEAD = 3 };
enum ParamKind { P_CONV = 0, P_BN_GAMMA = 1, P_BN_BETA = 2, P_FC_W = 3, P_BIAS = 4 };

struct ParamTensor {
  std::string name;
  int kind;
  int unit;
  int ndim;
  int64_t shape[5];
  int64_t numel;
  int64_t canon_off;  // offset in the canonical flat array (== internal master offset)
};

struct Unit {
  int kind;
  int cin, cout, stride;
  Dims in, out;
  Dims conv;   // stem: conv output dims before the pool
  Dims mask;   // att: mask-branch dims
  bool pool = false;
};

struct NetModel {
  rn_net_desc desc;
  std::vector<Unit> units;
  std::vector<ParamTensor> params;
  int64_t n_params = 0;
  int64_t n_bn_channels = 0;
  std::vector<int64_t> unit_costs;
  std::vector<int> part_first;  // size n_parts + 1
  std::vector<int64_t> part_loads;
  // index of first param tensor of each unit, and one-past-last
  std::vector<int> unit_param_begin, unit_param_end;
};

// Throws std::invalid_argument on a bad description.
NetModel build_net(const rn_net_desc &d);

void partition_units(const std::vector<int64_t> &costs, double alpha, int64_t max_merge_load,
                     std::vector<int> &first, std::vector<int64_t> &loads);

// f2 step-time model and contiguous split (sim.cpp)
void simulate_step(const rn_sim_desc &d, double *step, double *pipe, double *ar, double *stage_t);
void contiguous_split(int n, const int64_t *loads, int S, int32_t *genes, int64_t *max_load);

}  // namespace rn
