// net.cpp — 3D-ResAttNet structure, parameter layout, unit costs and the
// partitioning rule.  PAPER.md:364-366 (§4.3.1: Conv blocks = 3x3x3 conv + BN +
// ReLU; residual layer = two Conv blocks; residual self-attention block; conv
// complexity O(Co*Ci*T*H*W*Kt*Kh*Kw)), §3.1.1 P:154-156 (partitions are
// contiguous layer ranges, highly functional layers alone).  Readings X1-X11, G1.
#include "net.h"

#include <stdexcept>

namespace rn {

static void add_param(NetModel &m, const std::string &name, int kind, int unit,
                      std::initializer_list<int64_t> shape) {
  ParamTensor t;
  t.name = name;
  t.kind = kind;
  t.unit = unit;
  t.ndim = (int)shape.size();
  int i = 0;
  t.numel = 1;
  for (auto s : shape) {
    t.shape[i++] = s;
    t.numel *= s;
  }
  for (; i < 5; ++i) t.shape[i] = 1;
  t.canon_off = m.n_params;
  m.n_params += t.numel;
  if (kind == P_BN_GAMMA) m.n_bn_channels += t.numel;
  m.params.push_back(t);
}

static void add_block_params(NetModel &m, const std::string &pre, int unit, int cin, int cout, int stride) {
  add_param(m, pre + ".conv1", P_CONV, unit, {cout, cin, 3, 3, 3});
  add_param(m, pre + ".bn1.gamma", P_BN_GAMMA, unit, {cout});
  add_param(m, pre + ".bn1.beta", P_BN_BETA, unit, {cout});
  add_param(m, pre + ".conv2", P_CONV, unit, {cout, cout, 3, 3, 3});
  add_param(m, pre + ".bn2.gamma", P_BN_GAMMA, unit, {cout});
  add_param(m, pre + ".bn2.beta", P_BN_BETA, unit, {cout});
  if (stride != 1 || cin != cout) {
    add_param(m, pre + ".proj", P_CONV, unit, {cout, cin, 1, 1, 1});
    add_param(m, pre + ".projbn.gamma", P_BN_GAMMA, unit, {cout});
    add_param(m, pre + ".projbn.beta", P_BN_BETA, unit, {cout});
  }
}

// Per-sample MACs (P:366 conv complexity; light-layer constants SPEC S:87:
// BN 2, ReLU/pool/add/mul/sigmoid/upsample 1 per output element, GAP 1 per
// input element, FC in*out, softmax 2 per class).
static int64_t block_cost(int cin, int cout, int stride, Dims in) {
  Dims o = conv_out(in, 3, stride, 1);
  int64_t v = o.vol(), e = (int64_t)cout * v;
  int64_t c = (int64_t)cout * cin * v * 27 + 2 * e + e + (int64_t)cout * cout * v * 27 + 2 * e;
  if (stride != 1 || cin != cout) c += (int64_t)cout * cin * v + 2 * e;
  c += e + e;
  return c;
}

void partition_units(const std::vector<int64_t> &costs, double alpha, int64_t max_merge_load,
                     std::vector<int> &first, std::vector<int64_t> &loads) {
  const int n = (int)costs.size();
  first.clear();
  loads.clear();
  int64_t sum = 0;
  for (auto c : costs) sum += c;
  const double mean = (double)sum / (double)n;
  std::vector<char> heavy(n);
  for (int i = 0; i < n; ++i) heavy[i] = (double)costs[i] >= alpha * mean;
  int i = 0;
  while (i < n) {
    if (heavy[i]) {
      first.push_back(i);
      loads.push_back(costs[i]);
      ++i;
      continue;
    }
    int start = i;
    int64_t acc = 0;
    while (i < n && !heavy[i]) {
      if (max_merge_load > 0 && i > start && acc + costs[i] > max_merge_load) {
        first.push_back(start);
        loads.push_back(acc);
        start = i;
        acc = 0;
      }
      acc += costs[i];
      ++i;
    }
    first.push_back(start);
    loads.push_back(acc);
  }
  first.push_back(n);
}

NetModel build_net(const rn_net_desc &d) {
  NetModel m;
  m.desc = d;
  int stem_stride;
  bool stem_pool;
  std::vector<int> blocks, att_after;
  if (d.depth == 0) {
    stem_stride = 1; stem_pool = false; blocks = {1}; att_after = {0};
  } else if (d.depth == 18) {
    stem_stride = 2; stem_pool = true; blocks = {2, 2, 2, 2}; att_after = {0, 1, 2};
  } else if (d.depth == 34) {
    stem_stride = 2; stem_pool = true; blocks = {3, 4, 6, 3}; att_after = {0, 1, 2};
  } else {
    throw std::invalid_argument("depth must be 0 (tiny), 18 or 34");
  }
  if (d.base_width < 1 || d.base_width % 8 != 0 || d.base_width > 512)
    throw std::invalid_argument("base_width must be a positive multiple of 8, <= 512");
  if (d.in_d < 4 || d.in_h < 4 || d.in_w < 4 || d.in_d > 512 || d.in_h > 512 || d.in_w > 512)
    throw std::invalid_argument("input dims out of range [4, 512]");
  if (d.n_classes != 2) throw std::invalid_argument("n_classes must be 2 (P:360)");
  if (!(d.alpha > 0)) throw std::invalid_argument("alpha must be > 0");

  Dims in{d.in_d, d.in_h, d.in_w};
  Unit stem;
  stem.kind = U_STEM;
  stem.cin = 1;
  stem.cout = d.base_width;
  stem.stride = stem_stride;
  stem.in = in;
  stem.conv = conv_out(in, 3, stem_stride, 1);
  stem.pool = stem_pool;
  stem.out = stem_pool ? conv_out(stem.conv, 3, 2, 1) : stem.conv;
  m.units.push_back(stem);
  int c = d.base_width;
  Dims cur = stem.out;
  for (size_t si = 0; si < blocks.size(); ++si) {
    int width = d.base_width << si;
    for (int bi = 0; bi < blocks[si]; ++bi) {
      Unit u;
      u.kind = U_BLOCK;
      u.cin = c;
      u.cout = width;
      u.stride = (si > 0 && bi == 0) ? 2 : 1;
      u.in = cur;
      u.out = conv_out(cur, 3, u.stride, 1);
      m.units.push_back(u);
      c = width;
      cur = u.out;
    }
    bool att = false;
    for (int a : att_after) att |= (a == (int)si);
    if (att) {
      Unit u;
      u.kind = U_ATT;
      u.cin = u.cout = c;
      u.stride = 1;
      u.in = u.out = cur;
      u.mask = conv_out(cur, 3, 2, 1);
      m.units.push_back(u);
    }
  }
  Unit head;
  head.kind = U_HEAD;
  head.cin = c;
  head.cout = d.n_classes;
  head.stride = 1;
  head.in = cur;
  head.out = Dims{1, 1, 1};
  m.units.push_back(head);
  if ((int)m.units.size() > RN_MAX_UNITS) throw std::invalid_argument("too many units");
  for (auto &u : m.units)
    if (u.out.d < 1 || u.out.h < 1 || u.out.w < 1) throw std::invalid_argument("volume too small");

  // parameters, canonical order
  for (int ui = 0; ui < (int)m.units.size(); ++ui) {
    const Unit &u = m.units[ui];
    std::string p = "u" + std::to_string(ui);
    m.unit_param_begin.push_back((int)m.params.size());
    if (u.kind == U_STEM) {
      add_param(m, p + ".conv", P_CONV, ui, {u.cout, 1, 3, 3, 3});
      add_param(m, p + ".bn.gamma", P_BN_GAMMA, ui, {u.cout});
      add_param(m, p + ".bn.beta", P_BN_BETA, ui, {u.cout});
    } else if (u.kind == U_BLOCK) {
      add_block_params(m, p, ui, u.cin, u.cout, u.stride);
    } else if (u.kind == U_ATT) {
      add_block_params(m, p + ".trunk", ui, u.cout, u.cout, 1);
      add_block_params(m, p + ".mask", ui, u.cout, u.cout, 1);
      add_param(m, p + ".mconv1", P_CONV, ui, {u.cout, u.cout, 1, 1, 1});
      add_param(m, p + ".mbn.gamma", P_BN_GAMMA, ui, {u.cout});
      add_param(m, p + ".mbn.beta", P_BN_BETA, ui, {u.cout});
      add_param(m, p + ".mconv2", P_CONV, ui, {u.cout, u.cout, 1, 1, 1});
      add_param(m, p + ".mconv2.bias", P_BIAS, ui, {u.cout});
    } else {
      add_param(m, p + ".fc.weight", P_FC_W, ui, {u.cout, u.cin});
      add_param(m, p + ".fc.bias", P_BIAS, ui, {u.cout});
    }
    m.unit_param_end.push_back((int)m.params.size());
  }

  // unit costs (a1)
  for (const Unit &u : m.units) {
    int64_t cost = 0;
    if (u.kind == U_STEM) {
      int64_t v = u.conv.vol(), e = (int64_t)u.cout * v;
      cost = (int64_t)u.cout * v * 27 + 2 * e + e;
      if (u.pool) cost += (int64_t)u.cout * u.out.vol();
    } else if (u.kind == U_BLOCK) {
      cost = block_cost(u.cin, u.cout, u.stride, u.in);
    } else if (u.kind == U_ATT) {
      int64_t ch = u.cout, e = ch * u.in.vol();
      cost = block_cost(u.cout, u.cout, 1, u.in);
      cost += ch * u.mask.vol();
      cost += block_cost(u.cout, u.cout, 1, u.mask);
      cost += e;
      cost += ch * ch * u.in.vol() + 2 * e + e;
      cost += ch * ch * u.in.vol();
      cost += e + e;
    } else {
      cost = (int64_t)u.cin * u.in.vol() + (int64_t)u.cin * u.cout + 2 * u.cout;
    }
    m.unit_costs.push_back(cost);
  }
  partition_units(m.unit_costs, d.alpha, d.max_merge_load, m.part_first, m.part_loads);
  return m;
}

}  // namespace rn
