// tuckerplan (B200 engine) : multiplication trees — drop-in for reference ttm_tree.hpp:27-187.
// The value types are the reference's (nodes stored parent-first, children in insertion order = execution order);
// validation / canonical form / depth forward to the C ABI on flat kind/mode/parent arrays.
#pragma once

#include <vector>

#include "problem.hpp"

namespace tuckerplan {

enum class NodeKind { root, mode, leaf };

struct TreeNode {
  NodeKind kind;
  int mode = -1;
  int parent = -1;
  std::vector<int> children;
};

struct TtmTree {
  int n_modes = 0;
  std::vector<TreeNode> nodes;

  int add_node(NodeKind kind, int mode, int parent) {
    const int id = static_cast<int>(nodes.size());
    nodes.push_back(TreeNode{kind, mode, parent, {}});
    if (parent >= 0) nodes[parent].children.push_back(id);
    return id;
  }
  void pop_node() {
    const int parent = nodes.back().parent;
    if (parent >= 0) nodes[parent].children.pop_back();
    nodes.pop_back();
  }
  bool is_internal(int id) const { return nodes[id].kind == NodeKind::mode; }
  bool is_leaf(int id) const { return nodes[id].kind == NodeKind::leaf; }
};

inline TtmTree make_tree(int n_modes) {
  TtmTree t;
  t.n_modes = n_modes;
  t.add_node(NodeKind::root, -1, -1);
  return t;
}

namespace detail {
struct FlatTree {
  std::vector<int> kind, mode, parent;
  int size() const { return static_cast<int>(kind.size()); }
};
// The C ABI derives child order from stored order; a tree whose child lists disagree with its parent links or are
// not in ascending id order cannot be expressed and is rejected here the way the reference rejects it.
inline FlatTree flatten(const TtmTree& t) {
  FlatTree f;
  for (const TreeNode& n : t.nodes) {
    f.kind.push_back(static_cast<int>(n.kind));
    f.mode.push_back(n.mode);
    f.parent.push_back(n.parent);
  }
  for (int id = 0; id < f.size(); ++id) {
    int prev = id;
    for (int c : t.nodes[id].children) {
      if (c <= prev || c >= f.size() || t.nodes[c].parent != id) fail(Errc::bad_tree, "parent link mismatch");
      prev = c;
    }
  }
  return f;
}
inline TtmTree unflatten(int n_modes, const std::vector<int>& kind, const std::vector<int>& mode,
                         const std::vector<int>& parent, int count) {
  TtmTree t;
  t.n_modes = n_modes;
  for (int i = 0; i < count; ++i) t.add_node(static_cast<NodeKind>(kind[i]), mode[i], parent[i]);
  return t;
}
template <class Fn>
TtmTree tree_from_abi(int n_modes, Fn&& fn) {
  std::vector<int> kind(64), mode(64), parent(64);
  int count = 0;
  int status = fn(static_cast<int>(kind.size()), kind.data(), mode.data(), parent.data(), &count);
  if (status == TP_ERR_CAPACITY) {
    kind.resize(count), mode.resize(count), parent.resize(count);
    status = fn(count, kind.data(), mode.data(), parent.data(), &count);
  }
  check(status);
  return unflatten(n_modes, kind, mode, parent, count);
}
}  // namespace detail

inline void validate_tree(const TtmTree& t, const ProblemSpec& s) {
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  if (t.nodes.empty() || t.nodes[0].kind != NodeKind::root || t.nodes[0].parent != -1)
    fail(Errc::bad_tree, "node 0 must be the root");
  const detail::FlatTree f = detail::flatten(t);
  detail::check(tp_validate_tree(s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(),
                                 f.parent.data()));
}
inline bool is_canonical(const TtmTree& t) {
  const detail::FlatTree f = detail::flatten(t);
  int out = 0;
  detail::check(tp_tree_is_canonical(f.size(), f.kind.data(), f.mode.data(), f.parent.data(), &out));
  return out != 0;
}
inline TtmTree canonicalize(const TtmTree& t) {
  const detail::FlatTree f = detail::flatten(t);
  return detail::tree_from_abi(t.n_modes, [&](int cap, int* k, int* m, int* p, int* n) {
    return tp_canonicalize(t.n_modes, f.size(), f.kind.data(), f.mode.data(), f.parent.data(), cap, k, m, p, n);
  });
}
inline int tree_depth(const TtmTree& t) {
  const detail::FlatTree f = detail::flatten(t);
  int out = 0;
  detail::check(tp_tree_depth(f.size(), f.kind.data(), f.mode.data(), f.parent.data(), &out));
  return out;
}

}  // namespace tuckerplan
