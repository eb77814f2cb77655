// Host-side prerequisites of the hot path (kept on the CPU by design,
// SURVEY.md §2 "host prereq"): shear/postorder flattening into sf_problem rows
// and the seeded synthetic instance generator.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "sf_common.hpp"
#include "stripefrac_host.h"

using sf::set_error;

namespace {

// Children in node-index order, as finalize_topology builds them
// (newick.cpp:169-186). Returns the root, or -1 on malformed input.
int build_children(int32_t n, const int32_t* parent, std::vector<int64_t>& ptr,
                   std::vector<int32_t>& kids) {
  ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  int root = -1;
  for (int i = 0; i < n; ++i) {
    const int p = parent[i];
    if (p < 0) {
      if (root >= 0) {
        set_error("tree has more than one root");
        return -1;
      }
      root = i;
    } else {
      if (p >= n) {
        set_error("parent index out of range");
        return -1;
      }
      ++ptr[static_cast<std::size_t>(p) + 1];
    }
  }
  if (root < 0) {
    set_error("tree has no root");
    return -1;
  }
  for (int i = 0; i < n; ++i) ptr[static_cast<std::size_t>(i) + 1] += ptr[static_cast<std::size_t>(i)];
  kids.assign(static_cast<std::size_t>(n > 0 ? n - 1 : 0), 0);
  std::vector<int64_t> at(ptr.begin(), ptr.end() - 1);
  for (int i = 0; i < n; ++i)
    if (parent[i] >= 0) kids[static_cast<std::size_t>(at[static_cast<std::size_t>(parent[i])]++)] = i;
  return root;
}

}  // namespace

extern "C" sf_status sfh_flatten(int32_t n_nodes, const int32_t* parent, const double* length,
                                 int32_t n_features, const int32_t* feature_leaf,
                                 int32_t* n_rows, int32_t* parent_row, double* lengths,
                                 int32_t* leaf_feature) {
  if (n_nodes < 1 || !parent || !length || !feature_leaf || !n_rows || !parent_row ||
      !lengths || !leaf_feature || n_features < 1) {
    set_error("sfh_flatten: bad arguments");
    return SF_EINVAL;
  }
  std::vector<int64_t> ptr;
  std::vector<int32_t> kids;
  const int root = build_children(n_nodes, parent, ptr, kids);
  if (root < 0) return SF_EINVAL;
  auto n_kids = [&](int v) { return ptr[static_cast<std::size_t>(v) + 1] - ptr[static_cast<std::size_t>(v)]; };

  std::vector<int32_t> feat_of(static_cast<std::size_t>(n_nodes), -1);
  int n_leaves = 0;
  for (int i = 0; i < n_nodes; ++i) n_leaves += n_kids(i) == 0 ? 1 : 0;
  for (int f = 0; f < n_features; ++f) {
    const int leaf = feature_leaf[f];
    if (leaf < 0 || leaf >= n_nodes || n_kids(leaf) != 0) {
      set_error("table feature " + std::to_string(f) + " is not a leaf of the tree");
      return SF_EINVAL;
    }
    if (feat_of[static_cast<std::size_t>(leaf)] >= 0) {
      set_error("two table features map to the same leaf");
      return SF_EINVAL;
    }
    feat_of[static_cast<std::size_t>(leaf)] = f;
  }

  // kept[v]: v is a feature leaf or an ancestor of one (newick.cpp:318-323)
  const bool shear = n_features != n_leaves;  // embed.cpp:13
  std::vector<char> kept(static_cast<std::size_t>(n_nodes), 1);
  if (shear) {
    std::fill(kept.begin(), kept.end(), 0);
    for (int i = 0; i < n_nodes; ++i)
      if (feat_of[static_cast<std::size_t>(i)] >= 0)
        for (int v = i; v >= 0 && !kept[static_cast<std::size_t>(v)]; v = parent[v]) kept[static_cast<std::size_t>(v)] = 1;
  }
  auto live_count = [&](int v, int* only) {
    int c = 0;
    for (int64_t e = ptr[static_cast<std::size_t>(v)]; e < ptr[static_cast<std::size_t>(v) + 1]; ++e)
      if (kept[static_cast<std::size_t>(kids[static_cast<std::size_t>(e)])]) {
        ++c;
        *only = kids[static_cast<std::size_t>(e)];
      }
    return c;
  };

  // Rebuild the (sheared) tree in preorder, as rebuild_sheared does
  // (newick.cpp:288-307): a non-root node with exactly one live child is
  // folded into that child, carrying ((0 + l_top) + l_next) + ... and the
  // surviving node gets length + carry. Without shear nothing folds.
  struct NewNode {
    int32_t orig;
    int32_t parent;
    double length;
  };
  std::vector<NewNode> nn;
  nn.reserve(static_cast<std::size_t>(n_nodes));
  struct Frame {
    int32_t node;
    int32_t new_parent;
  };
  std::vector<Frame> stack;
  stack.push_back({root, -1});
  std::vector<int32_t> order;  // scratch for reversing children
  while (!stack.empty()) {
    const Frame f = stack.back();
    stack.pop_back();
    int node = f.node;
    double carry = 0.0;
    if (shear) {
      int only = -1;
      while (node != root && live_count(node, &only) == 1) {
        carry = carry + length[node];
        node = only;
      }
    }
    const int id = static_cast<int>(nn.size());
    nn.push_back({node, f.new_parent, node == root ? 0.0 : length[node] + carry});
    order.clear();
    for (int64_t e = ptr[static_cast<std::size_t>(node)]; e < ptr[static_cast<std::size_t>(node) + 1]; ++e)
      if (kept[static_cast<std::size_t>(kids[static_cast<std::size_t>(e)])]) order.push_back(kids[static_cast<std::size_t>(e)]);
    for (auto it = order.rbegin(); it != order.rend(); ++it) stack.push_back({*it, id});
  }

  // Postorder of the rebuilt tree, root excluded (newick.cpp:189-206).
  const int m = static_cast<int>(nn.size());
  std::vector<int64_t> cptr(static_cast<std::size_t>(m) + 1, 0);
  for (int i = 1; i < m; ++i) ++cptr[static_cast<std::size_t>(nn[static_cast<std::size_t>(i)].parent) + 1];
  for (int i = 0; i < m; ++i) cptr[static_cast<std::size_t>(i) + 1] += cptr[static_cast<std::size_t>(i)];
  std::vector<int32_t> ckids(static_cast<std::size_t>(m > 0 ? m - 1 : 0));
  {
    std::vector<int64_t> at(cptr.begin(), cptr.end() - 1);
    for (int i = 1; i < m; ++i)
      ckids[static_cast<std::size_t>(at[static_cast<std::size_t>(nn[static_cast<std::size_t>(i)].parent)]++)] = i;
  }
  std::vector<int32_t> row_of(static_cast<std::size_t>(m), -1);
  std::vector<std::pair<int32_t, int64_t>> st;
  st.emplace_back(0, cptr[0]);
  int32_t rows = 0;
  while (!st.empty()) {
    auto& [v, next] = st.back();
    if (next < cptr[static_cast<std::size_t>(v) + 1]) {
      const int32_t c = ckids[static_cast<std::size_t>(next++)];
      st.emplace_back(c, cptr[static_cast<std::size_t>(c)]);
    } else {
      if (v != 0) {
        const NewNode& nd = nn[static_cast<std::size_t>(v)];
        row_of[static_cast<std::size_t>(v)] = rows;
        lengths[rows] = nd.length;
        const bool leaf = cptr[static_cast<std::size_t>(v) + 1] == cptr[static_cast<std::size_t>(v)];
        leaf_feature[rows] = leaf ? feat_of[static_cast<std::size_t>(nd.orig)] : -1;
        if (leaf && leaf_feature[rows] < 0) {
          set_error("tree leaves and table features differ");
          return SF_EINVAL;
        }
        ++rows;
      }
      st.pop_back();
    }
  }
  for (int v = 1; v < m; ++v) {
    const int p = nn[static_cast<std::size_t>(v)].parent;
    parent_row[row_of[static_cast<std::size_t>(v)]] = p == 0 ? -1 : row_of[static_cast<std::size_t>(p)];
  }
  if (rows < 1) {
    set_error("tree has no rows after shearing");
    return SF_EINVAL;
  }
  *n_rows = rows;
  return SF_OK;
}

// ---------------------------------------------------------------- synth
// Restatement of random_tree / random_table / random_instance
// (synth.cpp:8-83) on the same <random> engines and distributions, so an
// instance is the reference's instance bit for bit (same libstdc++).
struct sfh_instance {
  std::vector<int32_t> parent;
  std::vector<double> length;
  std::vector<int32_t> feature_leaf;
  std::vector<int64_t> feat_ptr;
  std::vector<int32_t> sample_idx;
  std::vector<double> counts;
  std::vector<double> totals;
  int32_t n_samples = 0;
};

extern "C" sfh_instance* sfh_random_instance(uint64_t seed, int32_t n_samples, int32_t n_leaves,
                                             double density, int32_t table_features) {
  if (n_leaves < 1 || n_samples < 1) {
    set_error("random_instance: need at least one leaf and one sample");
    return nullptr;
  }
  try {
    auto inst = std::make_unique<sfh_instance>();
    std::mt19937_64 rng(seed);
    // random_tree (synth.cpp:8-40)
    const int total = 2 * n_leaves - 1;
    inst->parent.assign(static_cast<std::size_t>(total), -1);
    inst->length.assign(static_cast<std::size_t>(total), 0.0);
    std::vector<int> roots;
    roots.reserve(static_cast<std::size_t>(n_leaves));
    for (int f = 0; f < n_leaves; ++f) roots.push_back(f);
    std::uniform_real_distribution<double> len(0.0, 2.0);
    int next = n_leaves;
    while (roots.size() > 1) {
      std::uniform_int_distribution<std::size_t> pick(0, roots.size() - 1);
      const std::size_t ia = pick(rng);
      std::swap(roots[ia], roots.back());
      const int a = roots.back();
      roots.pop_back();
      std::uniform_int_distribution<std::size_t> pick2(0, roots.size() - 1);
      const std::size_t ib = pick2(rng);
      std::swap(roots[ib], roots.back());
      const int b = roots.back();
      roots.pop_back();
      const int join = next++;
      inst->parent[static_cast<std::size_t>(a)] = join;
      inst->length[static_cast<std::size_t>(a)] = len(rng);
      inst->parent[static_cast<std::size_t>(b)] = join;
      inst->length[static_cast<std::size_t>(b)] = len(rng);
      roots.push_back(join);
    }
    // features = leaf_names (node order f0..f{F-1}); shuffled subset (synth.cpp:75-80)
    std::vector<int32_t> features(static_cast<std::size_t>(n_leaves));
    for (int f = 0; f < n_leaves; ++f) features[static_cast<std::size_t>(f)] = f;
    if (table_features > 0 && table_features < n_leaves) {
      std::shuffle(features.begin(), features.end(), rng);
      features.resize(static_cast<std::size_t>(table_features));
    }
    inst->feature_leaf = features;
    // random_table (synth.cpp:42-68)
    const std::size_t F = features.size();
    std::vector<std::vector<std::pair<int32_t, double>>> entries(F);
    std::uniform_real_distribution<double> hit(0.0, 1.0);
    std::uniform_real_distribution<double> count(0.5, 64.0);
    std::uniform_int_distribution<std::size_t> any(0, F - 1);
    for (int s = 0; s < n_samples; ++s) {
      bool nonempty = false;
      for (std::size_t f = 0; f < F; ++f) {
        if (hit(rng) < density) {
          entries[f].emplace_back(s, count(rng));
          nonempty = true;
        }
      }
      if (!nonempty) entries[any(rng)].emplace_back(s, count(rng));
    }
    inst->n_samples = n_samples;
    inst->feat_ptr.assign(F + 1, 0);
    for (std::size_t f = 0; f < F; ++f) inst->feat_ptr[f + 1] = inst->feat_ptr[f] + static_cast<int64_t>(entries[f].size());
    inst->sample_idx.reserve(static_cast<std::size_t>(inst->feat_ptr[F]));
    inst->counts.reserve(static_cast<std::size_t>(inst->feat_ptr[F]));
    inst->totals.assign(static_cast<std::size_t>(n_samples), 0.0);
    for (std::size_t f = 0; f < F; ++f)
      for (const auto& [s, c] : entries[f]) {
        inst->sample_idx.push_back(s);
        inst->counts.push_back(c);
        inst->totals[static_cast<std::size_t>(s)] += c;  // synth.cpp:64-66
      }
    return inst.release();
  } catch (const std::exception& e) {
    set_error(std::string("random_instance: ") + e.what());
    return nullptr;
  }
}

extern "C" void sfh_instance_free(sfh_instance* inst) { delete inst; }
extern "C" int32_t sfh_instance_n_nodes(const sfh_instance* i) { return static_cast<int32_t>(i->parent.size()); }
extern "C" int32_t sfh_instance_n_samples(const sfh_instance* i) { return i->n_samples; }
extern "C" int32_t sfh_instance_n_features(const sfh_instance* i) { return static_cast<int32_t>(i->feature_leaf.size()); }
extern "C" int64_t sfh_instance_nnz(const sfh_instance* i) { return i->feat_ptr.back(); }
extern "C" const int32_t* sfh_instance_parent(const sfh_instance* i) { return i->parent.data(); }
extern "C" const double* sfh_instance_length(const sfh_instance* i) { return i->length.data(); }
extern "C" const int32_t* sfh_instance_feature_leaf(const sfh_instance* i) { return i->feature_leaf.data(); }
extern "C" const int64_t* sfh_instance_feat_ptr(const sfh_instance* i) { return i->feat_ptr.data(); }
extern "C" const int32_t* sfh_instance_sample_idx(const sfh_instance* i) { return i->sample_idx.data(); }
extern "C" const double* sfh_instance_counts(const sfh_instance* i) { return i->counts.data(); }
extern "C" const double* sfh_instance_sample_totals(const sfh_instance* i) { return i->totals.data(); }

extern "C" uint64_t sfh_fnv1a64(const void* data, uint64_t len, uint64_t h) {
  const auto* b = static_cast<const unsigned char*>(data);
  for (uint64_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
