// Host-side prerequisites of the hot path (kept on the CPU by design,
// SURVEY.md §2 "host prereq"): shear/postorder flattening into sf_problem rows
// and the seeded synthetic instance generator.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
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

// Row blocks formatted in parallel (std::to_chars with a precision is
// printf's "%.*g" in the C locale, without the locale and varargs cost),
// written in row order; memory stays bounded at one round of blocks.
extern "C" sf_status sfh_write_tsv(const char* path, int32_t n, const char* const* ids, const double* values,
                                   int32_t digits, int32_t threads) {
  if (!path || n < 0 || (n > 0 && (!ids || !values)) || digits < 1 || digits > 17)
    return set_error("write_tsv: bad arguments"), SF_EINVAL;
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return set_error(std::string("cannot open '") + path + "' for writing"), SF_EINVAL;
  struct Closer {
    std::FILE* f;
    ~Closer() {
      if (f) std::fclose(f);
    }
  } closer{f};
  std::string head;
  for (int32_t j = 0; j < n; ++j) {
    if (j) head.push_back('\t');
    head += ids[j];
  }
  head.push_back('\n');
  if (std::fwrite(head.data(), 1, head.size(), f) != head.size())
    return set_error(std::string("failed writing '") + path + "'"), SF_EINVAL;
  const unsigned T = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
  const int32_t rows_per_block = std::max<int32_t>(1, static_cast<int32_t>((8u << 20) / (static_cast<uint64_t>(n) * 24 + 1)));
  // two sets of row-block buffers: the threads format round r + 1 while
  // this thread writes round r
  std::vector<std::string> buf[2] = {std::vector<std::string>(T), std::vector<std::string>(T)};
  auto format = [&](std::string& out, int32_t r0, int32_t r1) {
    out.clear();
    char tmp[64];
    for (int32_t i = r0; i < r1; ++i) {
      out += ids[i];
      const double* row = values + static_cast<int64_t>(i) * n;
      for (int32_t j = 0; j < n; ++j) {
        tmp[0] = '\t';
        const auto res = std::to_chars(tmp + 1, tmp + sizeof(tmp), row[j], std::chars_format::general, digits);
        out.append(tmp, static_cast<std::size_t>(res.ptr - tmp));
      }
      out.push_back('\n');
    }
  };
  const int64_t round_rows = static_cast<int64_t>(T) * rows_per_block;
  auto launch = [&](int64_t r, std::vector<std::string>& set, std::vector<std::thread>& pool) {
    for (unsigned t = 0; t < T; ++t) {
      const int64_t a = r + static_cast<int64_t>(t) * rows_per_block;
      if (a >= n) {
        set[t].clear();
        continue;
      }
      const int64_t b = std::min<int64_t>(n, a + rows_per_block);
      pool.emplace_back(format, std::ref(set[t]), static_cast<int32_t>(a), static_cast<int32_t>(b));
    }
  };
  std::vector<std::thread> cur, next;
  if (n > 0) launch(0, buf[0], cur);
  int which = 0;
  for (int64_t r = 0; r < n; r += round_rows) {
    for (auto& th : cur) th.join();
    cur.clear();
    if (r + round_rows < n) launch(r + round_rows, buf[which ^ 1], next);
    bool ok = true;
    for (unsigned t = 0; t < T && ok; ++t)
      ok = std::fwrite(buf[which][t].data(), 1, buf[which][t].size(), f) == buf[which][t].size();
    if (!ok) {
      for (auto& th : next) th.join();
      return set_error(std::string("failed writing '") + path + "'"), SF_EINVAL;
    }
    std::swap(cur, next);
    which ^= 1;
  }
  if (std::fclose(f) != 0) {
    closer.f = nullptr;
    return set_error(std::string("failed writing '") + path + "'"), SF_EINVAL;
  }
  closer.f = nullptr;
  return SF_OK;
}

// ---- sparse table loader (table.cpp:105-168) ------------------------------------

struct sfh_table {
  std::vector<std::string> sample_ids, feature_ids;
  std::vector<int64_t> feat_ptr;
  std::vector<int32_t> sample_idx;
  std::vector<double> counts, totals;
};

namespace {

struct ParseError {
  int64_t line = -1;  // -1: none
  std::string msg;
};

struct Chunk {
  const char* begin;
  const char* end;
  int64_t first_line;  // 1-based number of the chunk's first line
  // parsed triplets: local feature id, sample (local id, or global when pinned), value
  std::vector<int32_t> f, s;
  std::vector<double> v;
  std::vector<std::string_view> feats, samples;  // local ids in first-appearance order
  ParseError err;
};

// The reference's parse_count on one cell: whole cell, finite, >= 0.
bool parse_value(std::string_view cell, double& v, std::string& msg, int64_t line) {
  v = 0.0;
  const auto res = std::from_chars(cell.data(), cell.data() + cell.size(), v);
  if (res.ec != std::errc() || res.ptr != cell.data() + cell.size()) {
    msg = "line " + std::to_string(line) + ": bad count '" + std::string(cell) + "'";
    return false;
  }
  if (!std::isfinite(v)) {
    msg = "line " + std::to_string(line) + ": count must be finite";
    return false;
  }
  if (v < 0.0) {
    msg = "line " + std::to_string(line) + ": count must be non-negative";
    return false;
  }
  return true;
}

void parse_chunk(Chunk& c, const std::unordered_map<std::string_view, int32_t>* pinned) {
  std::unordered_map<std::string_view, int32_t> fmap, smap;
  int64_t line = c.first_line;
  for (const char* p = c.begin; p < c.end; ++line) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(c.end - p)));
    const char* e = nl ? nl : c.end;
    std::string_view ln(p, static_cast<size_t>(e - p));
    p = nl ? nl + 1 : c.end;
    if (!ln.empty() && ln.back() == '\r') ln.remove_suffix(1);
    if (ln.empty()) continue;
    const size_t t1 = ln.find('\t');
    const size_t t2 = t1 == std::string_view::npos ? t1 : ln.find('\t', t1 + 1);
    if (t2 == std::string_view::npos || ln.find('\t', t2 + 1) != std::string_view::npos) {
      c.err = {line, "line " + std::to_string(line) + ": expected feature<TAB>sample<TAB>value"};
      return;
    }
    const std::string_view fid = ln.substr(0, t1), sid = ln.substr(t1 + 1, t2 - t1 - 1), val = ln.substr(t2 + 1);
    if (fid.empty()) {
      c.err = {line, "line " + std::to_string(line) + ": feature id is empty"};
      return;
    }
    if (sid.empty()) {
      c.err = {line, "line " + std::to_string(line) + ": sample id is empty"};
      return;
    }
    double v;
    std::string msg;
    if (!parse_value(val, v, msg, line)) {
      c.err = {line, msg};
      return;
    }
    int32_t s;
    if (pinned) {
      const auto it = pinned->find(sid);
      if (it == pinned->end()) {
        c.err = {line, "line " + std::to_string(line) + ": sample '" + std::string(sid) + "' not in the #samples header"};
        return;
      }
      s = it->second;
    } else {
      const auto it = smap.try_emplace(sid, static_cast<int32_t>(c.samples.size()));
      if (it.second) c.samples.push_back(sid);
      s = it.first->second;
    }
    const auto fit = fmap.try_emplace(fid, static_cast<int32_t>(c.feats.size()));
    if (fit.second) c.feats.push_back(fid);
    c.f.push_back(fit.first->second);
    c.s.push_back(s);
    c.v.push_back(v);
  }
}

}  // namespace

extern "C" sf_status sfh_load_table_sparse(const char* path, int32_t threads, sfh_table** out) {
  if (!path || !out) return set_error("load_table: bad arguments"), SF_EINVAL;
  const bool dbg = std::getenv("SF_DEBUG") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "stripefrac: load_table %s %.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tick).count());
    tick = now;
  };
  *out = nullptr;
  const std::string where = std::string(path) + ": ";
  std::FILE* fh = std::fopen(path, "rb");
  if (!fh) return set_error(std::string("cannot open table file '") + path + "'"), SF_EINVAL;
  std::string text;
  {
    std::fseek(fh, 0, SEEK_END);
    const long size = std::ftell(fh);
    std::fseek(fh, 0, SEEK_SET);
    text.resize(size > 0 ? static_cast<size_t>(size) : 0);
    const size_t got = text.empty() ? 0 : std::fread(&text[0], 1, text.size(), fh);
    std::fclose(fh);
    if (got != text.size()) return set_error(std::string("cannot read table file '") + path + "'"), SF_EINVAL;
  }
  phase("read");
  const char* p = text.data();
  const char* end = p + text.size();
  auto t = std::make_unique<sfh_table>();
  // the first non-empty line may be the "#samples" header
  int64_t line = 1;
  std::unordered_map<std::string_view, int32_t> pinned_map;
  bool pinned = false;
  const char* body = p;
  int64_t body_line = 1;
  for (const char* q = p; q < end; ++line) {
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(end - q)));
    const char* e = nl ? nl : end;
    std::string_view ln(q, static_cast<size_t>(e - q));
    if (!ln.empty() && ln.back() == '\r') ln.remove_suffix(1);
    if (ln.empty()) {
      q = nl ? nl + 1 : end;
      continue;
    }
    const size_t t1 = ln.find('\t');
    if (ln.substr(0, t1) == "#samples") {
      if (t1 == std::string_view::npos) return set_error(where + "#samples header names no samples"), SF_EINVAL;
      std::string_view rest = ln.substr(t1 + 1);
      for (;;) {
        const size_t tb = rest.find('\t');
        const std::string_view id = rest.substr(0, tb);
        if (id.empty()) return set_error(where + "sample id is empty"), SF_EINVAL;
        if (!pinned_map.emplace(id, static_cast<int32_t>(t->sample_ids.size())).second)
          return set_error(where + "duplicate sample id '" + std::string(id) + "'"), SF_EINVAL;
        t->sample_ids.emplace_back(id);
        if (tb == std::string_view::npos) break;
        rest = rest.substr(tb + 1);
      }
      pinned = true;
      body = nl ? nl + 1 : end;
      body_line = line + 1;
    } else {
      body = q;
      body_line = line;
    }
    break;
  }
  // chunks of whole lines, each with its first line number
  const unsigned T = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
  std::vector<Chunk> chunks;
  {
    const size_t len = static_cast<size_t>(end - body);
    const char* a = body;
    for (unsigned i = 0; i < T && a < end; ++i) {
      const char* b = i + 1 == T ? end : std::min(end, body + len * (i + 1) / T);
      if (b < end) {
        const char* nl = static_cast<const char*>(std::memchr(b, '\n', static_cast<size_t>(end - b)));
        b = nl ? nl + 1 : end;
      }
      if (b <= a) continue;
      chunks.push_back(Chunk{a, b, 0, {}, {}, {}, {}, {}, {}});
      a = b;
    }
    std::vector<int64_t> nls(chunks.size(), 0);
    std::vector<std::thread> pool;
    for (size_t i = 0; i < chunks.size(); ++i)
      pool.emplace_back([&, i] { nls[i] = std::count(chunks[i].begin, chunks[i].end, '\n'); });
    for (auto& th : pool) th.join();
    int64_t ln = body_line;
    for (size_t i = 0; i < chunks.size(); ++i) {
      chunks[i].first_line = ln;
      ln += nls[i];
    }
  }
  {
    std::vector<std::thread> pool;
    for (auto& c : chunks) pool.emplace_back(parse_chunk, std::ref(c), pinned ? &pinned_map : nullptr);
    for (auto& th : pool) th.join();
  }
  phase("parse");
  for (const auto& c : chunks)  // the first error in file order
    if (c.err.line >= 0) return set_error(where + c.err.msg), SF_EINVAL;
  // samples in first-appearance order (or the header's), features in byte order
  std::vector<std::vector<int32_t>> smap(chunks.size()), fmap(chunks.size());
  std::unordered_map<std::string_view, int32_t> gsamp, gfeat;
  std::vector<std::string_view> feats;
  for (size_t i = 0; i < chunks.size(); ++i) {
    auto& c = chunks[i];
    if (!pinned)
      for (const auto& sid : c.samples) {
        const auto it = gsamp.try_emplace(sid, static_cast<int32_t>(t->sample_ids.size()));
        if (it.second) t->sample_ids.emplace_back(sid);
        smap[i].push_back(it.first->second);
      }
    for (const auto& fid : c.feats) {
      const auto it = gfeat.try_emplace(fid, static_cast<int32_t>(feats.size()));
      if (it.second) feats.push_back(fid);
      fmap[i].push_back(it.first->second);
    }
  }
  if (t->sample_ids.empty()) return set_error(where + "sparse table names no samples"), SF_EINVAL;
  phase("merge ids");
  const int32_t F = static_cast<int32_t>(feats.size());
  std::vector<int32_t> order(static_cast<size_t>(F)), rank(static_cast<size_t>(F));
  for (int32_t i = 0; i < F; ++i) order[static_cast<size_t>(i)] = i;
  std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return feats[x] < feats[y]; });
  for (int32_t r = 0; r < F; ++r) rank[static_cast<size_t>(order[static_cast<size_t>(r)])] = r;
  // triplets bucketed by feature rank, file order kept (counting sort)
  std::vector<int64_t> off(static_cast<size_t>(F) + 1, 0);
  for (size_t i = 0; i < chunks.size(); ++i)
    for (const int32_t lf : chunks[i].f) ++off[static_cast<size_t>(rank[static_cast<size_t>(fmap[i][static_cast<size_t>(lf)])]) + 1];
  for (int32_t r = 0; r < F; ++r) off[static_cast<size_t>(r) + 1] += off[static_cast<size_t>(r)];
  std::vector<int32_t> bs(static_cast<size_t>(off.back()));
  std::vector<double> bv(static_cast<size_t>(off.back()));
  {
    std::vector<int64_t> at(off.begin(), off.end() - 1);
    for (size_t i = 0; i < chunks.size(); ++i) {
      const auto& c = chunks[i];
      for (size_t k = 0; k < c.f.size(); ++k) {
        const int32_t r = rank[static_cast<size_t>(fmap[i][static_cast<size_t>(c.f[k])])];
        const int64_t pos = at[static_cast<size_t>(r)]++;
        bs[static_cast<size_t>(pos)] = pinned ? c.s[k] : smap[i][static_cast<size_t>(c.s[k])];
        bv[static_cast<size_t>(pos)] = c.v[k];
      }
    }
  }
  chunks.clear();
  phase("sort features + bucket");
  // per feature: samples ascending, duplicates summed in file order
  // (std::map<int, double>::operator[] += v from 0.0), zero sums dropped
  std::vector<int64_t> kept(static_cast<size_t>(F) + 1, 0);
  {
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < T; ++w)
      pool.emplace_back([&, w] {
        std::vector<std::pair<int32_t, double>> seg;
        for (int32_t r = static_cast<int32_t>(w); r < F; r += static_cast<int32_t>(T)) {
          const int64_t a = off[static_cast<size_t>(r)], b = off[static_cast<size_t>(r) + 1];
          seg.clear();
          for (int64_t k = a; k < b; ++k) seg.emplace_back(bs[static_cast<size_t>(k)], bv[static_cast<size_t>(k)]);
          std::stable_sort(seg.begin(), seg.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
          int64_t o = a;
          for (size_t k = 0; k < seg.size();) {
            double sum = 0.0;
            const int32_t s = seg[k].first;
            for (; k < seg.size() && seg[k].first == s; ++k) sum += seg[k].second;
            if (sum > 0.0) {
              bs[static_cast<size_t>(o)] = s;
              bv[static_cast<size_t>(o)] = sum;
              ++o;
            }
          }
          kept[static_cast<size_t>(r) + 1] = o - a;
        }
      });
    for (auto& th : pool) th.join();
  }
  phase("per-feature sort + sums");
  t->feat_ptr.assign(static_cast<size_t>(F) + 1, 0);
  for (int32_t r = 0; r < F; ++r) t->feat_ptr[static_cast<size_t>(r) + 1] = t->feat_ptr[static_cast<size_t>(r)] + kept[static_cast<size_t>(r) + 1];
  t->sample_idx.resize(static_cast<size_t>(t->feat_ptr.back()));
  t->counts.resize(static_cast<size_t>(t->feat_ptr.back()));
  t->feature_ids.reserve(static_cast<size_t>(F));
  for (int32_t r = 0; r < F; ++r) {
    t->feature_ids.emplace_back(feats[static_cast<size_t>(order[static_cast<size_t>(r)])]);
    const int64_t a = off[static_cast<size_t>(r)];
    std::copy(bs.begin() + a, bs.begin() + a + kept[static_cast<size_t>(r) + 1],
              t->sample_idx.begin() + t->feat_ptr[static_cast<size_t>(r)]);
    std::copy(bv.begin() + a, bv.begin() + a + kept[static_cast<size_t>(r) + 1],
              t->counts.begin() + t->feat_ptr[static_cast<size_t>(r)]);
  }
  // check_sample_totals (table.cpp:55-62): summed in feature order
  t->totals.assign(t->sample_ids.size(), 0.0);
  for (size_t k = 0; k < t->sample_idx.size(); ++k) t->totals[static_cast<size_t>(t->sample_idx[k])] += t->counts[k];
  for (size_t s = 0; s < t->totals.size(); ++s)
    if (!(t->totals[s] > 0.0)) return set_error(where + "sample '" + t->sample_ids[s] + "' has no counts"), SF_EINVAL;
  phase("csr + totals");
  *out = t.release();
  return SF_OK;
}

extern "C" void sfh_table_free(sfh_table* t) { delete t; }
extern "C" int32_t sfh_table_n_samples(const sfh_table* t) { return static_cast<int32_t>(t->sample_ids.size()); }
extern "C" int32_t sfh_table_n_features(const sfh_table* t) { return static_cast<int32_t>(t->feature_ids.size()); }
extern "C" int64_t sfh_table_nnz(const sfh_table* t) { return t->feat_ptr.back(); }
extern "C" const char* sfh_table_sample_id(const sfh_table* t, int32_t i) { return t->sample_ids[static_cast<size_t>(i)].c_str(); }
extern "C" const char* sfh_table_feature_id(const sfh_table* t, int32_t i) { return t->feature_ids[static_cast<size_t>(i)].c_str(); }
extern "C" const int64_t* sfh_table_feat_ptr(const sfh_table* t) { return t->feat_ptr.data(); }
extern "C" const int32_t* sfh_table_sample_idx(const sfh_table* t) { return t->sample_idx.data(); }
extern "C" const double* sfh_table_counts(const sfh_table* t) { return t->counts.data(); }
extern "C" const double* sfh_table_sample_totals(const sfh_table* t) { return t->totals.data(); }
