// Host planner for the HOOI hot path: problem spec, product trees, the
// load-optimal tree search, exact MAC accounting, processor grids and the
// volume-optimal static grid.  Everything is exact u64 arithmetic and every
// SELECTION (tree shape, node ids, grid) is bit-identical to the reference's,
// because the executor's buffer sizes, launch order and the partitioner's cut
// points all derive from it.
//
// Reference behaviour followed (paths under reference proj/include/tuckerplan):
//   problem.hpp:37-86, ttm_tree.hpp:36-187, tree_cost.hpp:25-63,
//   tree_opt.hpp:56-150 (tie rules :13-15), tree_builders.hpp:27-91,
//   grid.hpp:36-125, grid_volume.hpp:32-110.
#pragma once

#include <array>
#include <algorithm>
#include <future>
#include <numeric>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.hpp"

namespace tpb {

constexpr int kMaxModes = TP_MAX_MODES;
constexpr u64 kMaxElements = u64{1} << 62;  // problem.hpp:22

struct Spec {
  std::vector<u64> L, K;
  int n() const { return static_cast<int>(L.size()); }
};

inline Spec make_spec(int n, const u64* L, const u64* K) {
  if (n < 0 || (n > 0 && (!L || !K))) raise(TP_ERR_BAD_DIMS, "spec needs matching non-empty L and K");
  Spec s;
  s.L.assign(L, L + n);
  s.K.assign(K, K + n);
  return s;
}

// problem.hpp:37-53
inline void validate_spec(const Spec& s) {
  const int n = s.n();
  if (n == 0 || s.K.size() != s.L.size()) raise(TP_ERR_BAD_DIMS, "spec needs matching non-empty L and K");
  if (n > kMaxModes) raise(TP_ERR_BAD_DIMS, "at most 16 modes supported");
  u64 total = 1;
  for (int m = 0; m < n; ++m) {
    if (s.L[m] == 0) raise(TP_ERR_BAD_DIMS, "zero length at mode " + std::to_string(m), m);
    if (s.K[m] < 1 || s.K[m] > s.L[m])
      raise(TP_ERR_K_TOO_LARGE, "K out of [1, L] at mode " + std::to_string(m), m);
    total = mul_or_throw(total, s.L[m]);
  }
  if (total > kMaxElements) raise(TP_ERR_OVERFLOW, "input exceeds 2^62 elements");
}

// problem.hpp:78-86: prod over modes of (K if multiplied else L)
inline u64 partial_cardinality(const Spec& s, std::uint32_t done) {
  u64 total = 1;
  for (int m = 0; m < s.n(); ++m) total = mul_or_throw(total, ((done >> m) & 1u) ? s.K[m] : s.L[m]);
  return total;
}

// ------------------------------------------------------------------- trees
struct Tree {
  int n_modes = 0;
  std::vector<int> kind, mode, parent;
  std::vector<std::vector<int>> kids;

  int size() const { return static_cast<int>(kind.size()); }
  bool internal(int id) const { return kind[id] == TP_NODE_MODE; }
  bool leaf(int id) const { return kind[id] == TP_NODE_LEAF; }

  int add(int k, int m, int p) {
    const int id = size();
    kind.push_back(k);
    mode.push_back(m);
    parent.push_back(p);
    kids.emplace_back();
    if (p >= 0) kids[p].push_back(id);
    return id;
  }
};

inline Tree new_tree(int n_modes) {
  Tree t;
  t.n_modes = n_modes;
  t.add(TP_NODE_ROOT, -1, -1);
  return t;
}

// Flat arrays (C ABI) -> Tree.  Child lists follow stored order, which is the
// reference's insertion order.  Links that cannot be represented are reported
// as bad_tree here; the structural rules are checked by validate_tree.
inline Tree tree_from_arrays(int n_modes, int n_nodes, const int* kind, const int* mode, const int* parent) {
  if (n_nodes < 0 || (n_nodes > 0 && (!kind || !mode || !parent))) raise(TP_ERR_BAD_TREE, "missing tree arrays");
  Tree t;
  t.n_modes = n_modes;
  t.kind.assign(kind, kind + n_nodes);
  t.mode.assign(mode, mode + n_nodes);
  t.parent.assign(parent, parent + n_nodes);
  t.kids.resize(n_nodes);
  for (int i = 0; i < n_nodes; ++i) {
    if (kind[i] < TP_NODE_ROOT || kind[i] > TP_NODE_LEAF) raise(TP_ERR_BAD_TREE, "unknown node kind");
    const int p = parent[i];
    if (i == 0) continue;  // checked by validate_tree
    if (p < 0 || p >= i) raise(TP_ERR_BAD_TREE, "nodes must be stored parent first");
    t.kids[p].push_back(i);
  }
  return t;
}

namespace detail {
inline std::uint32_t all_modes(int n) { return n >= 32 ? ~std::uint32_t{0} : ((std::uint32_t{1} << n) - 1); }

// ttm_tree.hpp:61-99: every root-to-leaf path for leaf n multiplies exactly the other modes, once each.
inline void walk_paths(const Tree& t, int id, std::uint32_t seen, std::vector<int>& leaf_seen) {
  const int kind = t.kind[id], m = t.mode[id];
  if (kind == TP_NODE_LEAF) {
    if (!t.kids[id].empty()) raise(TP_ERR_BAD_TREE, "leaf with children");
    if (m < 0 || m >= t.n_modes) raise(TP_ERR_BAD_TREE, "leaf mode out of range", m);
    if (leaf_seen[m]++) raise(TP_ERR_BAD_TREE, "duplicate leaf", m);
    if (seen != (all_modes(t.n_modes) & ~(std::uint32_t{1} << m)))
      raise(TP_ERR_BAD_TREE, "path to leaf " + std::to_string(m) + " does not cover the complementary modes", m);
    return;
  }
  if (kind == TP_NODE_MODE) {
    if (m < 0 || m >= t.n_modes) raise(TP_ERR_BAD_TREE, "label out of range", m);
    if ((seen >> m) & 1u) raise(TP_ERR_BAD_TREE, "mode repeated along a path", m);
    seen |= std::uint32_t{1} << m;
  }
  if (t.kids[id].empty()) raise(TP_ERR_BAD_TREE, "internal node without children");
  for (int c : t.kids[id]) walk_paths(t, c, seen, leaf_seen);
}
}  // namespace detail

// ttm_tree.hpp:103-119
inline void validate_tree(const Tree& t, const Spec& s) {
  if (t.n_modes != s.n()) raise(TP_ERR_SHAPE_MISMATCH, "tree and spec mode counts differ");
  if (t.size() == 0 || t.kind[0] != TP_NODE_ROOT || t.parent[0] != -1)
    raise(TP_ERR_BAD_TREE, "node 0 must be the root");
  for (int i = 1; i < t.size(); ++i) {
    if (t.kind[i] == TP_NODE_ROOT) raise(TP_ERR_BAD_TREE, "multiple roots");
    if (t.parent[i] < 0 || t.parent[i] >= i) raise(TP_ERR_BAD_TREE, "nodes must be stored parent first");
  }
  std::vector<int> leaf_seen(t.n_modes, 0);
  detail::walk_paths(t, 0, 0u, leaf_seen);
  for (int m = 0; m < t.n_modes; ++m)
    if (!leaf_seen[m]) raise(TP_ERR_BAD_TREE, "missing leaf", m);
}

// ttm_tree.hpp:123-135: no two mode children of one node share a label
inline bool is_canonical(const Tree& t) {
  for (int id = 0; id < t.size(); ++id) {
    std::uint32_t labels = 0;
    for (int c : t.kids[id]) {
      if (!t.internal(c)) continue;
      const std::uint32_t bit = std::uint32_t{1} << t.mode[c];
      if (labels & bit) return false;
      labels |= bit;
    }
  }
  return true;
}

namespace detail {
// ttm_tree.hpp:141-163: equal-labelled mode children of the merged sources are grouped in first-seen order.
inline void merge_into(const Tree& in, const std::vector<int>& sources, Tree& out, int dst) {
  std::vector<std::vector<int>> groups;
  for (int src : sources)
    for (int c : in.kids[src]) {
      std::vector<int>* home = nullptr;
      if (in.internal(c))
        for (auto& g : groups)
          if (in.internal(g.front()) && in.mode[g.front()] == in.mode[c]) {
            home = &g;
            break;
          }
      if (home)
        home->push_back(c);
      else
        groups.push_back({c});
    }
  for (const auto& g : groups) {
    const int head = g.front();
    const int id = out.add(in.kind[head], in.mode[head], dst);
    if (in.kind[head] != TP_NODE_LEAF) merge_into(in, g, out, id);
  }
}
}  // namespace detail

// ttm_tree.hpp:168-173
inline Tree canonicalize(const Tree& t) {
  Tree out = new_tree(t.n_modes);
  detail::merge_into(t, {0}, out, 0);
  return out;
}

// ttm_tree.hpp:176-187: longest run of mode nodes on any root-to-leaf path
inline int tree_depth(const Tree& t) {
  std::vector<int> depth(t.size(), 0);
  int best = 0;
  for (int id = 0; id < t.size(); ++id) {  // parent-first storage
    const int up = t.parent[id] >= 0 && t.parent[id] < id ? depth[t.parent[id]] : 0;
    depth[id] = up + (t.internal(id) ? 1 : 0);
    best = std::max(best, depth[id]);
  }
  return best;
}

// ------------------------------------------------------------------- costs
struct Cards {
  std::vector<u64> in, out;
};

// tree_cost.hpp:25-41
inline Cards node_cardinalities(const Tree& t, const Spec& s) {
  validate_tree(t, s);
  Cards c;
  c.in.resize(t.size());
  c.out.resize(t.size());
  const u64 total = partial_cardinality(s, 0);
  for (int id = 0; id < t.size(); ++id) {
    const u64 in = t.parent[id] < 0 ? total : c.out[t.parent[id]];
    c.in[id] = in;
    c.out[id] = t.internal(id) ? scale_exact(in, s.K[t.mode[id]], s.L[t.mode[id]]) : in;
  }
  return c;
}

struct Cost {
  u64 total_macs = 0;
  std::vector<u64> per_node;
  int n_internal = 0;
  int depth = 0;
};

// tree_cost.hpp:50-63
inline Cost tree_cost(const Tree& t, const Spec& s, Cards* cards_out = nullptr) {
  Cards cards = node_cardinalities(t, s);
  Cost r;
  r.per_node.assign(t.size(), 0);
  for (int id = 0; id < t.size(); ++id) {
    if (!t.internal(id)) continue;
    r.per_node[id] = mul_or_throw(s.K[t.mode[id]], cards.in[id]);
    r.total_macs = add_or_throw(r.total_macs, r.per_node[id]);
    ++r.n_internal;
  }
  r.depth = tree_depth(t);
  if (cards_out) *cards_out = std::move(cards);
  return r;
}

// Extents of the tensor a node PRODUCES: K on every mode multiplied on the path from the root, L elsewhere
// (simulate.hpp:62-67).
inline std::vector<u64> node_extents(const Tree& t, const Spec& s, int id) {
  std::vector<u64> ext = s.L;
  for (int at = id; at >= 0; at = t.parent[at])
    if (t.kind[at] == TP_NODE_MODE) ext[t.mode[at]] = s.K[t.mode[at]];
  return ext;
}

// ------------------------------------------------------- optimal tree search
// State (P, Q): P = modes already multiplied on the path, Q = outputs this subtree owes; R = rest.
//   finish(P,Q) = 0                                         |Q| = 1, R empty
//   reuse n in R: K_n |T[P]| + finish(P+n, Q)
//   split Q = Q1 + Q2 (Q1 holds Q's lowest mode): finish(P,Q1) + finish(P,Q2)
// Candidates are scanned reuse-first in ascending mode, then splits in ascending Q1 mask, and only a strictly
// smaller cost replaces the incumbent — the reference's tie rules (tree_opt.hpp:13-15, 70-92).
class TreeSearch {
 public:
  explicit TreeSearch(const Spec& s, bool reuse_greedy = false)
      : spec_(s), all_(detail::all_modes(s.n())), greedy_(reuse_greedy) {}

  struct Cell {
    u64 cost = 0;
    std::uint8_t move = 0;  // 0 finished, 1 reuse, 2 split
    std::uint8_t reuse_mode = 0;
    std::uint16_t q1 = 0;
  };

  const Cell& finish(std::uint32_t p, std::uint32_t q) {
    const std::uint32_t key = p | (q << 16);
    if (auto it = memo_.find(key); it != memo_.end()) return it->second;
    const std::uint32_t r = all_ & ~p & ~q;
    Cell cell;
    if (__builtin_popcount(q) == 1 && r == 0) return memo_.emplace(key, cell).first->second;

    cell.cost = kSat;
    const u64 card = partial_cardinality(spec_, p);
    for (std::uint32_t left = r; left; left &= left - 1) {
      const int n = __builtin_ctz(left);
      const u64 c = add_sat(mul_sat(spec_.K[n], card), finish(p | (1u << n), q).cost);
      if (c < cell.cost) cell = Cell{c, 1, static_cast<std::uint8_t>(n), 0};
    }
    if (__builtin_popcount(q) >= 2 && (!greedy_ || r == 0)) {
      const std::uint32_t low = q & (~q + 1);
      const std::uint32_t rest = q & ~low;
      // proper subsets of `rest` in ascending numeric order (the full set would leave Q2 empty)
      for (std::uint32_t sub = 0; sub != rest; sub = (sub - rest) & rest) {
        const std::uint32_t q1 = sub | low;
        const u64 c = add_sat(finish(p, q1).cost, finish(p, q & ~q1).cost);
        if (c < cell.cost) cell = Cell{c, 2, 0, static_cast<std::uint16_t>(q1)};
      }
    }
    return memo_.emplace(key, cell).first->second;
  }

  // Emits the chosen subtree under `host`: Q1 side before Q2 side, so node ids are DFS preorder
  // (tree_opt.hpp:96-115).
  void emit(std::uint32_t p, std::uint32_t q, int host, Tree& t) {
    const Cell cell = finish(p, q);
    if (cell.move == 0) {
      t.add(TP_NODE_LEAF, __builtin_ctz(q), host);
    } else if (cell.move == 1) {
      const int v = t.add(TP_NODE_MODE, cell.reuse_mode, host);
      emit(p | (1u << cell.reuse_mode), q, v, t);
    } else {
      emit(p, cell.q1, host, t);
      emit(p, q & ~static_cast<std::uint32_t>(cell.q1), host, t);
    }
  }

  std::size_t states() const { return memo_.size(); }
  std::uint32_t all() const { return all_; }

 private:
  const Spec& spec_;
  std::uint32_t all_;
  bool greedy_;
  std::unordered_map<std::uint32_t, Cell> memo_;
};

struct OptimalTree {
  Tree tree;
  u64 total_macs = 0;
  std::size_t dp_states = 0;
};

// tree_opt.hpp:126-138
inline OptimalTree optimal_tree(const Spec& s) {
  validate_spec(s);
  TreeSearch search(s);
  const u64 cost = search.finish(0, search.all()).cost;
  if (cost == kSat) raise(TP_ERR_OVERFLOW, "optimal cost not representable in 64 bits");
  OptimalTree r;
  r.tree = new_tree(s.n());
  search.emit(0, search.all(), 0, r.tree);
  r.total_macs = cost;
  r.dp_states = search.states();
  return r;
}

// tree_opt.hpp:143-150
inline u64 reuse_greedy_cost(const Spec& s) {
  validate_spec(s);
  TreeSearch search(s, true);
  const u64 cost = search.finish(0, search.all()).cost;
  if (cost == kSat) raise(TP_ERR_OVERFLOW, "cost not representable in 64 bits");
  return cost;
}

// ------------------------------------------------------------ fixed builders
// tree_builders.hpp:27-47
inline std::vector<int> chain_order(const Spec& s, int order) {
  std::vector<int> modes(s.n());
  std::iota(modes.begin(), modes.end(), 0);
  if (order == TP_CHAIN_BY_COST) {
    std::stable_sort(modes.begin(), modes.end(), [&](int a, int b) { return s.K[a] < s.K[b]; });
  } else if (order == TP_CHAIN_BY_RATIO) {
    std::stable_sort(modes.begin(), modes.end(), [&](int a, int b) {
      return static_cast<unsigned __int128>(s.K[a]) * s.L[b] < static_cast<unsigned __int128>(s.K[b]) * s.L[a];
    });
  } else if (order != TP_CHAIN_INPUT) {
    raise(TP_ERR_BAD_ARGUMENT, "unknown chain order");
  }
  return modes;
}

// tree_builders.hpp:49-60: one private chain per output
inline Tree chain_tree(const Spec& s, int order = TP_CHAIN_INPUT) {
  validate_spec(s);
  const std::vector<int> seq = chain_order(s, order);
  Tree t = new_tree(s.n());
  for (int out = 0; out < s.n(); ++out) {
    int at = 0;
    for (int m : seq)
      if (m != out) at = t.add(TP_NODE_MODE, m, at);
    t.add(TP_NODE_LEAF, out, at);
  }
  return t;
}

namespace detail {
// tree_builders.hpp:66-81: halve the outputs; each half first multiplies the other half's modes
inline void balanced_below(Tree& t, const std::vector<int>& outs, int at) {
  if (outs.size() == 1) {
    t.add(TP_NODE_LEAF, outs[0], at);
    return;
  }
  const std::size_t half = (outs.size() + 1) / 2;
  const std::vector<int> lo(outs.begin(), outs.begin() + half), hi(outs.begin() + half, outs.end());
  int a = at;
  for (int m : hi) a = t.add(TP_NODE_MODE, m, a);
  balanced_below(t, lo, a);
  int b = at;
  for (int m : lo) b = t.add(TP_NODE_MODE, m, b);
  balanced_below(t, hi, b);
}
}  // namespace detail

// tree_builders.hpp:85-91
inline Tree balanced_tree(const Spec& s) {
  validate_spec(s);
  std::vector<int> outs(s.n());
  std::iota(outs.begin(), outs.end(), 0);
  Tree t = new_tree(s.n());
  detail::balanced_below(t, outs, 0);
  return t;
}

// bench.hpp:128-137
inline Tree build_tree(const Spec& s, int strategy) {
  switch (strategy) {
    case TP_TREE_CHAIN_INPUT: return chain_tree(s, TP_CHAIN_INPUT);
    case TP_TREE_CHAIN_BY_COST: return chain_tree(s, TP_CHAIN_BY_COST);
    case TP_TREE_CHAIN_BY_RATIO: return chain_tree(s, TP_CHAIN_BY_RATIO);
    case TP_TREE_BALANCED: return balanced_tree(s);
    case TP_TREE_OPTIMAL: return optimal_tree(s).tree;
  }
  raise(TP_ERR_BAD_ARGUMENT, "unknown strategy");
}

// hooi.hpp:163-183: per leaf mode, the modes along its private root chain
inline std::vector<std::vector<int>> chain_paths(const Tree& t) {
  std::vector<std::vector<int>> paths(t.n_modes);
  std::vector<char> seen(t.n_modes, 0);
  for (int c : t.kids[0]) {
    std::vector<int> modes;
    int at = c;
    while (t.kind[at] == TP_NODE_MODE) {
      modes.push_back(t.mode[at]);
      if (t.kids[at].size() != 1) raise(TP_ERR_NEEDS_CHAIN_TREE, "tree is not a chain scheme");
      at = t.kids[at][0];
    }
    if (t.kind[at] != TP_NODE_LEAF || seen[t.mode[at]]) raise(TP_ERR_NEEDS_CHAIN_TREE, "tree is not a chain scheme");
    seen[t.mode[at]] = 1;
    paths[t.mode[at]] = std::move(modes);
  }
  for (char s : seen)
    if (!s) raise(TP_ERR_NEEDS_CHAIN_TREE, "tree is not a chain scheme");
  return paths;
}

// -------------------------------------------------------------------- grids
using Grid = std::vector<u64>;

// grid.hpp:36-45
inline void validate_grid(const Grid& q, const Spec& s, u64 procs) {
  if (static_cast<int>(q.size()) != s.n()) raise(TP_ERR_INVALID_GRID, "grid and spec mode counts differ");
  u64 prod = 1;
  for (int m = 0; m < s.n(); ++m)
    if (q[m] < 1 || q[m] > s.K[m])
      raise(TP_ERR_INVALID_GRID, "grid extent outside [1, K] at mode " + std::to_string(m), m);
  for (u64 v : q) prod = mul_or_throw(prod, v);
  if (prod != procs) raise(TP_ERR_INVALID_GRID, "grid does not multiply out to the processor count");
}

// grid.hpp:49-70: psi(P,N) = prod over prime powers p^e of C(e+N-1, N-1)
inline u64 grid_count(u64 procs, int n_modes) {
  if (procs == 0 || n_modes < 1) raise(TP_ERR_BAD_ARGUMENT, "need procs >= 1 and modes >= 1");
  auto binom = [](u64 n, u64 k) {
    u64 r = 1;
    for (u64 i = 1; i <= k; ++i) r = mul_or_throw(r, n - k + i) / i;
    return r;
  };
  u64 count = 1, rem = procs;
  for (u64 p = 2; p <= rem / p; ++p) {
    u64 e = 0;
    while (rem % p == 0) {
      rem /= p;
      ++e;
    }
    if (e) count = mul_or_throw(count, binom(e + n_modes - 1, n_modes - 1));
  }
  if (rem > 1) count = mul_or_throw(count, static_cast<u64>(n_modes));
  return count;
}

// grid.hpp:96-111: every q with prod q = P and q_n <= K_n, lexicographic
inline std::vector<Grid> enumerate_grids(u64 procs, const Spec& s) {
  validate_spec(s);
  if (procs == 0) raise(TP_ERR_BAD_ARGUMENT, "need procs >= 1");
  std::vector<u64> divs;
  for (u64 d = 1; d <= procs / d; ++d)
    if (procs % d == 0) {
      divs.push_back(d);
      if (d != procs / d) divs.push_back(procs / d);
    }
  std::sort(divs.begin(), divs.end());
  std::vector<Grid> out;
  Grid cur(s.n(), 1);
  const int last = s.n() - 1;
  // iterative odometer over divisor choices for modes 0..N-2; the last mode takes the remainder
  struct Frame {
    std::size_t next;
    u64 rem;
  };
  std::vector<Frame> stack{{0, procs}};
  while (!stack.empty()) {
    const int m = static_cast<int>(stack.size()) - 1;
    Frame& f = stack.back();
    if (m == last) {
      if (f.rem <= s.K[m]) {
        cur[m] = f.rem;
        out.push_back(cur);
      }
      stack.pop_back();
      continue;
    }
    bool descended = false;
    while (f.next < divs.size()) {
      const u64 d = divs[f.next++];
      if (d > s.K[m]) {
        f.next = divs.size();
        break;
      }
      if (f.rem % d) continue;
      cur[m] = d;
      stack.push_back({0, f.rem / d});
      descended = true;
      break;
    }
    if (!descended) stack.pop_back();
  }
  return out;
}

// grid.hpp:114-119: floor cut points
inline std::vector<u64> block_bounds(u64 len, u64 parts) {
  if (parts == 0) raise(TP_ERR_BAD_ARGUMENT, "need parts >= 1");
  std::vector<u64> cuts(parts + 1);
  for (u64 b = 0; b <= parts; ++b) cuts[b] = static_cast<u64>(static_cast<unsigned __int128>(b) * len / parts);
  return cuts;
}

// grid.hpp:122-125
inline u64 block_of(u64 c, u64 len, u64 parts) {
  if (len == 0) raise(TP_ERR_BAD_ARGUMENT, "need len >= 1");
  return static_cast<u64>((static_cast<unsigned __int128>(c) * parts + parts - 1) / len);
}

struct Volume {
  u64 total = 0;
  std::vector<u64> per_node;  // indexed by node id, 0 for root/leaves
};

namespace detail {
inline Volume volume_under(const Tree& t, const Cards& cards, const Grid& q) {
  Volume v;
  v.per_node.assign(t.size(), 0);
  for (int id = 0; id < t.size(); ++id) {
    if (!t.internal(id)) continue;
    v.per_node[id] = mul_or_throw(q[t.mode[id]] - 1, cards.out[id]);
    v.total = add_or_throw(v.total, v.per_node[id]);
  }
  return v;
}
}  // namespace detail

// grid_volume.hpp:32-46: sum over TTM nodes of (q_n - 1) |Out_u|
inline Volume static_volume(const Tree& t, const Spec& s, const Grid& q, u64 procs) {
  validate_grid(q, s, procs);
  return detail::volume_under(t, node_cardinalities(t, s), q);
}

struct StaticGrid {
  Grid q;
  Volume volume;
};

// grid_volume.hpp:56-110: exhaustive scan, first minimum in lexicographic order; the threaded scan reduces
// chunk minima in grid order so the answer never depends on `threads`.
inline StaticGrid optimal_static_grid(const Tree& t, const Spec& s, u64 procs, int threads = 1) {
  const std::vector<Grid> grids = enumerate_grids(procs, s);
  if (grids.empty()) raise(TP_ERR_NO_VALID_GRID, "no grid with prod q = procs fits under K");
  const Cards cards = node_cardinalities(t, s);
  auto scan = [&](std::size_t lo, std::size_t hi) {
    std::pair<u64, std::size_t> best{detail::volume_under(t, cards, grids[lo]).total, lo};
    for (std::size_t i = lo + 1; i < hi; ++i) {
      const u64 v = detail::volume_under(t, cards, grids[i]).total;
      if (v < best.first) best = {v, i};
    }
    return best;
  };
  std::pair<u64, std::size_t> best;
  if (threads <= 1 || grids.size() < 2) {
    best = scan(0, grids.size());
  } else {
    const std::size_t chunk = (grids.size() + threads - 1) / threads;
    std::vector<std::future<std::pair<u64, std::size_t>>> parts;
    for (std::size_t lo = 0; lo < grids.size(); lo += chunk)
      parts.push_back(std::async(std::launch::async, scan, lo, std::min(lo + chunk, grids.size())));
    best = {kSat, 0};
    bool have = false;
    for (auto& p : parts) {
      const auto r = p.get();
      if (!have || r.first < best.first) {
        best = r;
        have = true;
      }
    }
  }
  return StaticGrid{grids[best.second], static_volume(t, s, grids[best.second], procs)};
}

// ---- per-node grids (grid_dynamic.hpp) -------------------------------------------------------------------
// A scheme gives the root an anchor grid and every TTM node its own; a node whose grid differs from its parent's
// first redistributes its whole input (|In_u| elements), then multiplies and pays (q_n - 1)|Out_u| as before.
struct Scheme {
  Grid root;
  std::vector<Grid> node;  // indexed by node id; empty for the root and the leaves
};

struct SchemeVolume {
  u64 total = 0;
  std::vector<u64> ttm, regrid;  // indexed by node id
};

inline const Grid& scheme_parent_grid(const Tree& t, const Scheme& sc, int id) {
  const int up = t.parent[id];
  return t.kind[up] == TP_NODE_ROOT ? sc.root : sc.node[up];
}

// grid_dynamic.hpp:37-62
inline SchemeVolume scheme_volume(const Tree& t, const Spec& s, const Scheme& sc, u64 procs) {
  validate_grid(sc.root, s, procs);
  const Cards cards = node_cardinalities(t, s);
  SchemeVolume v;
  v.ttm.assign(t.size(), 0);
  v.regrid.assign(t.size(), 0);
  for (int id = 0; id < t.size(); ++id) {
    if (!t.internal(id)) continue;
    if (id >= static_cast<int>(sc.node.size()) || sc.node[id].empty())
      raise(TP_ERR_MISSING_ASSIGNMENT, "no grid for internal node " + std::to_string(id));
    validate_grid(sc.node[id], s, procs);
    if (sc.node[id] != scheme_parent_grid(t, sc, id)) v.regrid[id] = cards.in[id];
    v.ttm[id] = mul_or_throw(sc.node[id][t.mode[id]] - 1, cards.out[id]);
    v.total = add_or_throw(v.total, add_or_throw(v.ttm[id], v.regrid[id]));
  }
  return v;
}

struct DynamicScheme {
  Scheme scheme;
  SchemeVolume volume;
};

// grid_dynamic.hpp:141-167.  below[u][g] = least volume of the subtree at TTM node u when its parent hands it grid
// g: either keep g, or pay |In_u| and switch to the node's best grid (found once per node: it does not depend on g).
// Ties keep the parent's grid, and among switch targets the first in enumeration order.  `legacy_target` ranks the
// switch targets by the children's volume alone (grid_dynamic.hpp:64-66, 107-109).
// Node ids grow from parent to child (ttm_tree.hpp:111-112), so one descending pass fills the table bottom-up and
// one ascending pass reads the choices back.
inline DynamicScheme optimal_dynamic_scheme(const Tree& t, const Spec& s, u64 procs, bool legacy_target = false) {
  const std::vector<Grid> grids = enumerate_grids(procs, s);
  if (grids.empty()) raise(TP_ERR_NO_VALID_GRID, "no grid with prod q = procs fits under K");
  const Cards cards = node_cardinalities(t, s);
  const std::size_t ng = grids.size();
  std::vector<std::vector<u64>> below(t.size());
  std::vector<u64> switch_cost(t.size(), 0);        // |In_u| + volume under the node's best grid
  std::vector<std::size_t> switch_to(t.size(), 0);
  auto kids_sum = [&](int id, std::size_t g) {
    u64 sum = 0;
    for (int c : t.kids[id])
      if (t.internal(c)) sum = add_or_throw(sum, below[c][g]);
    return sum;
  };
  auto own = [&](int id, std::size_t g) { return mul_or_throw(grids[g][t.mode[id]] - 1, cards.out[id]); };
  for (int id = t.size() - 1; id > 0; --id) {
    if (!t.internal(id)) continue;
    std::vector<u64> keep(ng);
    u64 best_rank = kSat;
    std::size_t arg = 0;
    for (std::size_t g = 0; g < ng; ++g) {
      const u64 kids = kids_sum(id, g);
      keep[g] = add_or_throw(own(id, g), kids);
      const u64 rank = legacy_target ? kids : keep[g];
      if (rank < best_rank) {
        best_rank = rank;
        arg = g;
      }
    }
    switch_to[id] = arg;
    switch_cost[id] = add_or_throw(cards.in[id], keep[arg]);
    below[id].resize(ng);
    for (std::size_t g = 0; g < ng; ++g) below[id][g] = std::min(keep[g], switch_cost[id]);
  }
  // the root's grid is free: it only anchors its children
  std::size_t root_g = 0;
  u64 best = kSat;
  for (std::size_t g = 0; g < ng; ++g) {
    const u64 v = kids_sum(0, g);
    if (v < best) {
      best = v;
      root_g = g;
    }
  }
  DynamicScheme out;
  out.scheme.root = grids[root_g];
  out.scheme.node.assign(t.size(), Grid{});
  std::vector<std::size_t> chosen(t.size(), root_g);
  for (int id = 1; id < t.size(); ++id) {
    if (!t.internal(id)) continue;
    const std::size_t from = chosen[t.parent[id]];
    const u64 keep = add_or_throw(own(id, from), kids_sum(id, from));
    chosen[id] = keep <= switch_cost[id] ? from : switch_to[id];
    out.scheme.node[id] = grids[chosen[id]];
  }
  out.volume = scheme_volume(t, s, out.scheme, procs);
  return out;
}

// simulate.hpp:104-121: elements of a tensor with extents `ext` whose owner rank changes between two grids.
// Counted per mode-wise overlap of the two block partitions instead of element by element.
inline u64 count_moved(const std::vector<u64>& ext, const Grid& from, const Grid& to) {
  const int n = static_cast<int>(ext.size());
  // stay[m][(a, b)] = coordinates of mode m that lie in block a of `from` and block b of `to`
  std::vector<std::vector<std::array<u64, 3>>> pieces(n);
  for (int m = 0; m < n; ++m) {
    const std::vector<u64> ca = block_bounds(ext[m], from[m]), cb = block_bounds(ext[m], to[m]);
    for (u64 a = 0; a < from[m]; ++a)
      for (u64 b = 0; b < to[m]; ++b) {
        const u64 lo = std::max(ca[a], cb[b]), hi = std::min(ca[a + 1], cb[b + 1]);
        if (hi > lo) pieces[m].push_back({a, b, hi - lo});
      }
  }
  u64 total = 1, same = 0;
  for (int m = 0; m < n; ++m) total = mul_or_throw(total, ext[m]);
  // walk the product of the per-mode pieces, accumulating both ranks
  std::vector<std::size_t> at(n, 0);
  for (int m = 0; m < n; ++m)
    if (pieces[m].empty()) return 0;
  while (true) {
    u64 ra = 0, rb = 0, elems = 1;
    for (int m = 0; m < n; ++m) {
      const auto& pc = pieces[m][at[m]];
      ra = ra * from[m] + pc[0];
      rb = rb * to[m] + pc[1];
      elems *= pc[2];
    }
    if (ra == rb) same += elems;
    int carry = n;
    while (carry > 0 && ++at[carry - 1] == pieces[carry - 1].size()) at[--carry] = 0;
    if (carry == 0) break;
  }
  return total - same;
}

}  // namespace tpb
