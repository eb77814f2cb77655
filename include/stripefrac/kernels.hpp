// Drop-in replacement for the reference's include/stripefrac/kernels.hpp
// (/root/reference/proj/include/stripefrac/kernels.hpp): same types, same
// entry points, same preconditions and error messages, same counter law —
// but every stripe update, finalize and condense runs on B200 through the C
// ABI in stripefrac_cuda.h (libstripefrac_cuda.so). Put this directory ahead
// of the reference's include directory; the rest of the reference library
// (newick, table, embed, stripes, validate, bench) is used unchanged.
//
// Semantics kept from the reference:
//  * compute_unifrac<Real> (kernels.hpp:268-316): precision/instantiation,
//    batch and step checks, stripe range checks (allocate_stripes), shear via
//    sheared_to_table, finalize, counters accumulated with +=;
//  * variant / batch_capacity / step_size / threads never change bits
//    (README.md:36-44); `threads` is accepted and ignored — stripes are
//    sharded over all visible sm_100 devices instead;
//  * accumulate (kernels.hpp:232-248) and finalize (:251-259) act on host
//    StripeSets, computing on device;
//  * compute_distance_matrix (:319-326) condenses on device.
// Unweighted results are the correctly rounded exact sums (fixed-point
// arithmetic, kernel 10): within ~1e-14 relative of the reference's
// sequential fp64 sums (gate: 1e-12). Weighted ones agree within 1e-12
// relative (fp64, FMA). Defining STRIPEFRAC_B200_EXACT selects the kernels
// that replay the reference's adds in the reference's order: bitwise
// identical for every metric.
#pragma once

#include <cstdint>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "stripefrac/common.hpp"
#include "stripefrac/embed.hpp"
#include "stripefrac/newick.hpp"
#include "stripefrac/stripes.hpp"
#include "stripefrac/table.hpp"
#include "stripefrac_cuda.h"

namespace stripefrac {

struct KernelConfig {
  Metric metric = Metric::Unweighted;
  Variant variant = Variant::Tiled;
  Precision precision = Precision::Fp64;
  int batch_capacity = 64;  // embedding rows per pass (accounting only here)
  int step_size = 0;        // sample tile width (accounting only here)

  int resolved_step_size() const {
    if (step_size > 0) return step_size;
    return precision == Precision::Fp32 ? 32 : 16;
  }
};

struct KernelCounters {
  std::uint64_t accumulator_writes = 0;
  std::uint64_t embedding_reads = 0;
  std::uint64_t kernel_passes = 0;

  KernelCounters& operator+=(const KernelCounters& o) {
    accumulator_writes += o.accumulator_writes;
    embedding_reads += o.embedding_reads;
    kernel_passes += o.kernel_passes;
    return *this;
  }
};

namespace b200 {

inline void check(sf_status st) {
  if (st != SF_OK) throw Error(sf_last_error());
}

inline sf_metric metric_code(Metric m) {
  switch (m) {
    case Metric::Unweighted: return SF_UNWEIGHTED;
    case Metric::WeightedUnnormalized: return SF_WEIGHTED_UNNORMALIZED;
    case Metric::WeightedNormalized: return SF_WEIGHTED_NORMALIZED;
  }
  throw Error("unknown metric");
}

template <class Real>
constexpr sf_precision precision_code() {
  return std::is_same_v<Real, float> ? SF_FP32 : SF_FP64;
}

inline sf_exec default_exec() {
  sf_exec ex{};
#ifdef STRIPEFRAC_B200_EXACT
  ex.flags = SF_EXEC_EXACT_NO_FMA;
#endif
  return ex;
}

// A sheared tree (leaf set == feature set) + table as sf_problem rows:
// rows in PhyloTree::postorder order (newick.cpp:189-206).
struct FlatProblem {
  std::vector<int32_t> parent_row, leaf_feature, sample_idx;
  std::vector<double> lengths, counts;
  std::vector<int64_t> feat_ptr;
  sf_problem p{};
};

inline void flatten(const PhyloTree& sheared, const SampleTable& table, FlatProblem& out) {
  std::unordered_map<std::string, int> feature_idx;
  for (int f = 0; f < table.n_features(); ++f)
    feature_idx.emplace(table.feature_ids[static_cast<std::size_t>(f)], f);
  const std::size_t E = sheared.postorder.size();
  std::vector<int32_t> row_of(static_cast<std::size_t>(sheared.n_nodes()), -1);
  for (std::size_t r = 0; r < E; ++r) row_of[static_cast<std::size_t>(sheared.postorder[r])] = static_cast<int32_t>(r);
  out.parent_row.resize(E);
  out.leaf_feature.resize(E);
  out.lengths.resize(E);
  for (std::size_t r = 0; r < E; ++r) {
    const int v = sheared.postorder[r];
    const TreeNode& nd = sheared.nodes[static_cast<std::size_t>(v)];
    out.parent_row[r] = nd.parent == sheared.root ? -1 : row_of[static_cast<std::size_t>(nd.parent)];
    out.lengths[r] = nd.length;
    if (sheared.is_leaf(v)) {
      auto it = feature_idx.find(nd.name);
      if (it == feature_idx.end())
        throw Error("tree leaf '" + nd.name + "' is not a table feature; shear the tree first");
      out.leaf_feature[r] = it->second;
    } else {
      out.leaf_feature[r] = -1;
    }
  }
  out.feat_ptr.assign(static_cast<std::size_t>(table.n_features()) + 1, 0);
  for (int f = 0; f < table.n_features(); ++f) {
    const auto& ent = table.entries[static_cast<std::size_t>(f)];
    out.feat_ptr[static_cast<std::size_t>(f) + 1] = out.feat_ptr[static_cast<std::size_t>(f)] + static_cast<int64_t>(ent.size());
    for (const auto& [s, c] : ent) {
      out.sample_idx.push_back(s);
      out.counts.push_back(c);
    }
  }
  out.p.n_rows = static_cast<int32_t>(E);
  out.p.parent_row = out.parent_row.data();
  out.p.lengths = out.lengths.data();
  out.p.leaf_feature = out.leaf_feature.data();
  out.p.n_samples = table.n_samples();
  out.p.n_features = table.n_features();
  out.p.feat_ptr = out.feat_ptr.data();
  out.p.sample_idx = out.sample_idx.data();
  out.p.counts = out.counts.data();
  out.p.sample_totals = table.sample_totals.data();
}

// counter law (kernels.hpp:202-207, 246, 292)
inline void count(KernelCounters& c, const KernelConfig& cfg, std::uint64_t rows,
                  std::uint64_t entries, std::uint64_t passes) {
  c.accumulator_writes += (cfg.variant == Variant::Naive ? rows : passes) * entries;
  c.embedding_reads += 2 * rows * entries;
  c.kernel_passes += passes;
}

}  // namespace b200

// Fold one host embedding batch into the stripe set on device. Counts one pass.
template <class Real>
void accumulate(StripeSet<Real>& set, const EmbeddingBatch<Real>& batch,
                const KernelConfig& cfg, KernelCounters& counters) {
  if (set.finalized) throw Error("cannot accumulate into a finalized stripe set");
  if (batch.filled < 1) throw Error("embedding batch is empty");
  if (batch.n_samples != set.n_samples)
    throw Error("batch and stripe set disagree on the sample count");
  if (batch.emb.rows() < batch.filled || batch.emb.cols() != batch.n_samples_padded)
    throw Error("embedding batch shape is inconsistent");
  if (cfg.metric != set.metric)
    throw Error("kernel metric does not match the stripe set");
  if (cfg.variant == Variant::Tiled &&
      batch.n_samples_padded % cfg.resolved_step_size() != 0)
    throw Error("batch padding is not a multiple of the step size");
  b200::check(sf_accumulate_batch(batch.emb.data(), batch.lengths.data(), batch.filled,
                                  set.n_samples, batch.n_samples_padded,
                                  b200::metric_code(set.metric), b200::precision_code<Real>(),
                                  set.start, set.stop, set.distances.data(),
                                  set.has_totals() ? set.totals.data() : nullptr, 0));
  const std::uint64_t entries = static_cast<std::uint64_t>(set.n_stripes()) *
                                static_cast<std::uint64_t>(set.n_samples);
  b200::count(counters, cfg, static_cast<std::uint64_t>(batch.filled), entries, 1);
}

// Divide distances by totals (0/0 -> 0) on device; flips `finalized`.
template <class Real>
void finalize(StripeSet<Real>& set) {
  if (set.finalized) throw Error("stripe set was already finalized");
  if (set.has_totals())
    b200::check(sf_finalize(b200::precision_code<Real>(), static_cast<int64_t>(set.distances.size()),
                            set.distances.data(), set.totals.data(), 0));
  set.finalized = true;
}

// End-to-end stripe computation on device: shear on host, embed + stripe
// update + finalize on every visible B200 (stripes sharded, no collective).
template <class Real>
StripeSet<Real> compute_unifrac(const PhyloTree& tree, const SampleTable& table,
                                const KernelConfig& cfg, int start = 0, int stop = -1,
                                int threads = 1, KernelCounters* counters_out = nullptr) {
  (void)threads;
  constexpr Precision kPrec =
      std::is_same_v<Real, float> ? Precision::Fp32 : Precision::Fp64;
  if (cfg.precision != kPrec)
    throw Error("config asks for " + std::string(name(cfg.precision)) +
                " but compute_unifrac was instantiated for " + std::string(name(kPrec)));
  if (cfg.batch_capacity < 1) throw Error("batch capacity must be >= 1");
  if (cfg.resolved_step_size() < 1) throw Error("step size must be >= 1");

  const int S = total_stripes(table.n_samples());
  if (stop < 0) stop = S;
  const PhyloTree sheared = sheared_to_table(tree, table);
  auto set = allocate_stripes<Real>(table.n_samples(), start, stop, cfg.metric);
  b200::FlatProblem flat;
  b200::flatten(sheared, table, flat);
  // the reference Embedder's checks (embed.cpp:17-40) apply to the flattened rows too
  if (table.n_features() != sheared.n_leaves())
    throw Error("tree leaves and table features differ; shear the tree first");
  const sf_exec ex = b200::default_exec();
  b200::check(sf_compute_stripes(&flat.p, b200::metric_code(cfg.metric), b200::precision_code<Real>(),
                                 set.start, set.stop, set.distances.data(),
                                 set.has_totals() ? set.totals.data() : nullptr, 1, &ex, nullptr));
  set.finalized = true;
  if (counters_out) {
    const std::uint64_t E = sheared.postorder.size();
    const std::uint64_t B = static_cast<std::uint64_t>(cfg.batch_capacity);
    b200::count(*counters_out, cfg, E,
                static_cast<std::uint64_t>(set.n_stripes()) * static_cast<std::uint64_t>(set.n_samples),
                (E + B - 1) / B);
  }
  return set;
}

// Full pipeline to a condensed matrix: the stripes never leave the device;
// condense runs there and the n x n matrix is copied into dm.values once.
template <class Real>
DistanceMatrix compute_distance_matrix(const PhyloTree& tree, const SampleTable& table,
                                       const KernelConfig& cfg, int threads = 1,
                                       KernelCounters* counters_out = nullptr) {
  (void)threads;
  constexpr Precision kPrec =
      std::is_same_v<Real, float> ? Precision::Fp32 : Precision::Fp64;
  if (cfg.precision != kPrec)
    throw Error("config asks for " + std::string(name(cfg.precision)) +
                " but compute_distance_matrix was instantiated for " + std::string(name(kPrec)));
  if (cfg.batch_capacity < 1) throw Error("batch capacity must be >= 1");
  if (cfg.resolved_step_size() < 1) throw Error("step size must be >= 1");
  const int n = table.n_samples();
  const int S = total_stripes(n);
  const PhyloTree sheared = sheared_to_table(tree, table);
  b200::FlatProblem flat;
  b200::flatten(sheared, table, flat);
  if (table.n_features() != sheared.n_leaves())
    throw Error("tree leaves and table features differ; shear the tree first");
  DistanceMatrix dm;
  dm.sample_ids = table.sample_ids;
  dm.precision = kPrec;
  dm.values.resize(n, n);  // every entry is written on device
  const sf_exec ex = b200::default_exec();
  const sf_status st = sf_compute_distance_matrix(&flat.p, b200::metric_code(cfg.metric),
                                                  b200::precision_code<Real>(), dm.values.data(), &ex, nullptr);
  if (st != SF_OK) {
    const std::string msg = sf_last_error();
    if (msg.find("duplicated") != std::string::npos)
      throw Error("condense: duplicated slot disagrees");
    throw Error(msg);
  }
  if (counters_out) {
    const std::uint64_t E = sheared.postorder.size();
    const std::uint64_t B = static_cast<std::uint64_t>(cfg.batch_capacity);
    b200::count(*counters_out, cfg, E, static_cast<std::uint64_t>(S) * static_cast<std::uint64_t>(n),
                (E + B - 1) / B);
  }
  return dm;
}

}  // namespace stripefrac
