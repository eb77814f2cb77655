/*
 * stripefrac_host.h — host-side prerequisites of the hot path, C ABI.
 *
 * Shear + postorder flattening of a tree into sf_problem rows, and the
 * reference's seeded synthetic instance generator (bit-identical streams), so
 * that the Python mirror and bench.py can build sf_problem inputs without the
 * reference library. Lives in the same shared object as stripefrac_cuda.h.
 */
#ifndef STRIPEFRAC_HOST_H_
#define STRIPEFRAC_HOST_H_

#include <stdint.h>

#include "stripefrac_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Flatten a rooted tree (parent[i] = -1 for the root only) against a table
 * whose feature f is leaf node feature_leaf[f]:
 *  - if every leaf is a table feature, the tree is used unchanged
 *    (embed.cpp:13), otherwise it is sheared to the feature leaves with
 *    unary chains collapsed by summing lengths (newick.cpp:288-331);
 *  - rows are the sheared tree's postorder without the root
 *    (newick.cpp:189-206), children visited in node-index order.
 * Outputs have capacity n_nodes; *n_rows receives E. parent_row[r] = -1 when
 * the parent is the root. Returns SF_EINVAL on malformed input.
 */
sf_status sfh_flatten(int32_t n_nodes, const int32_t* parent, const double* length,
                      int32_t n_features, const int32_t* feature_leaf, int32_t* n_rows,
                      int32_t* parent_row, double* lengths, int32_t* leaf_feature);

/*
 * random_instance(seed, n_samples, n_leaves, density, table_features)
 * (synth.cpp:70-83): node i < n_leaves is leaf "f<i>", internal nodes follow;
 * samples are "s<j>". The table's feature f is leaf node feature_leaf[f]
 * (a shuffled subset when 0 < table_features < n_leaves).
 */
typedef struct sfh_instance sfh_instance;
sfh_instance* sfh_random_instance(uint64_t seed, int32_t n_samples, int32_t n_leaves,
                                  double density, int32_t table_features);
void sfh_instance_free(sfh_instance* inst);
int32_t sfh_instance_n_nodes(const sfh_instance* inst);
int32_t sfh_instance_n_samples(const sfh_instance* inst);
int32_t sfh_instance_n_features(const sfh_instance* inst);
int64_t sfh_instance_nnz(const sfh_instance* inst);
const int32_t* sfh_instance_parent(const sfh_instance* inst);  /* [n_nodes] */
const double* sfh_instance_length(const sfh_instance* inst);   /* [n_nodes] */
const int32_t* sfh_instance_feature_leaf(const sfh_instance* inst); /* [F] */
const int64_t* sfh_instance_feat_ptr(const sfh_instance* inst);     /* [F+1] */
const int32_t* sfh_instance_sample_idx(const sfh_instance* inst);   /* [nnz] */
const double* sfh_instance_counts(const sfh_instance* inst);        /* [nnz] */
const double* sfh_instance_sample_totals(const sfh_instance* inst); /* [n] */

/* FNV-1a 64 over raw bytes, chainable (common.cpp:50-57); the .strf checksum. */
uint64_t sfh_fnv1a64(const void* data, uint64_t len, uint64_t h);

/*
 * write_tsv(path, dm) (stripes.cpp:311-340): the n x n row-major matrix as
 * the reference's TSV — a header of the ids, then per row its id and the
 * values with "%.<digits>g" (17 for fp64, 9 for fp32), tab-separated —
 * byte for byte, formatted by `threads` host threads (0 = all) in row blocks
 * written in order. Replaces the reference's single-threaded snprintf loop
 * (C3: 6.25e8 values, a 12.5 GB file).
 */
sf_status sfh_write_tsv(const char* path, int32_t n, const char* const* ids, const double* values,
                        int32_t digits, int32_t threads);

/*
 * load_table_file(path, TableFormat::TsvSparse) (table.cpp:105-168, 176-184):
 * feature<TAB>sample<TAB>value triplets, an optional leading "#samples"
 * header pinning the sample order (else first appearance), duplicates of a
 * (feature, sample) summed in file order, features in byte order, samples
 * ascending, zero sums dropped, totals summed in feature order — the same
 * table bit for bit, and the same first error ("<path>: line N: ..."), parsed
 * by `threads` host threads (0 = all) instead of one std::map insertion per
 * triplet. The table is an opaque handle read through the accessors below.
 */
typedef struct sfh_table sfh_table;
sf_status sfh_load_table_sparse(const char* path, int32_t threads, sfh_table** out);
void sfh_table_free(sfh_table* t);
int32_t sfh_table_n_samples(const sfh_table* t);
int32_t sfh_table_n_features(const sfh_table* t);
int64_t sfh_table_nnz(const sfh_table* t);
const char* sfh_table_sample_id(const sfh_table* t, int32_t i);
const char* sfh_table_feature_id(const sfh_table* t, int32_t i);
const int64_t* sfh_table_feat_ptr(const sfh_table* t);
const int32_t* sfh_table_sample_idx(const sfh_table* t);
const double* sfh_table_counts(const sfh_table* t);
const double* sfh_table_sample_totals(const sfh_table* t);

#ifdef __cplusplus
}
#endif

#endif /* STRIPEFRAC_HOST_H_ */
