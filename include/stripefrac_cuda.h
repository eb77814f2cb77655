/*
 * stripefrac_cuda.h — C ABI of the B200 (sm_100a) Striped-UniFrac hot path.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/include/stripefrac/kernels.hpp). Plain pointers and
 * sizes only; no CUDA, Eigen or torch types cross it. Every entry point
 * replaces one reference interface, cited per function below. The C++ header
 * include/stripefrac/kernels.hpp re-exposes the reference API on top of it.
 *
 * Conventions:
 *  - The caller owns every host buffer. Stripe outputs are row-major
 *    (stop-start) x n arrays of float (SF_FP32) or double (SF_FP64): exactly
 *    StripeSet::distances.data() / totals.data() (stripes.hpp:25-37).
 *  - The library owns device memory (per call, or per sf_plan).
 *  - No exceptions cross the ABI: functions return sf_status and the message
 *    of the last failure on this thread is sf_last_error().
 *  - There is no CPU fallback: with no usable sm_100 device every compute
 *    entry point fails with SF_ECUDA.
 */
#ifndef STRIPEFRAC_CUDA_H_
#define STRIPEFRAC_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 3

typedef enum sf_status {
  SF_OK = 0,
  SF_EINVAL = 1, /* bad argument / precondition (reference: throws stripefrac::Error) */
  SF_ENOMEM = 2, /* device or host allocation failed */
  SF_ECUDA = 3,  /* CUDA runtime failure, or no sm_100 device */
  SF_ESTATE = 4  /* object in the wrong state (e.g. already finalized) */
} sf_status;

/* Metric codes are the .strf metric codes (stripes.cpp:143-150). */
typedef enum sf_metric {
  SF_UNWEIGHTED = 1,
  SF_WEIGHTED_UNNORMALIZED = 2,
  SF_WEIGHTED_NORMALIZED = 3,
  /* Extension (not in the reference, parity unpinned): generalized UniFrac
   * with exponent sf_exec.alpha over the weighted embedding (Chen et al.
   * 2012, in Striped UniFrac's form); finalize divides d by t like WN. It
   * has no .strf code in the reference's format. */
  SF_GENERALIZED = 4
} sf_metric;

/* Precision codes are the scalar width in bytes (.strf byte 5). */
typedef enum sf_precision { SF_FP32 = 4, SF_FP64 = 8 } sf_precision;

/*
 * A sheared tree + sample table flattened into postorder rows. Row r is the
 * r-th non-root node of PhyloTree::postorder (newick.cpp:189-206) after
 * sheared_to_table (embed.cpp:8-15). Children of a row are the rows whose
 * parent_row is r, folded in increasing row order — the reference's fold
 * order (embed.cpp:71-79).
 */
typedef struct sf_problem {
  int32_t n_rows;              /* E >= 1 */
  const int32_t* parent_row;   /* [E]; -1 when the parent is the root; else > r */
  const double* lengths;       /* [E]; branch length above the row, finite, >= 0 */
  const int32_t* leaf_feature; /* [E]; table feature index for leaves, -1 for internal rows */
  int32_t n_samples;           /* n >= 2 */
  int32_t n_features;          /* F >= 1 */
  const int64_t* feat_ptr;     /* [F+1] CSR row pointers of the table, by feature */
  const int32_t* sample_idx;   /* [nnz] sample of each entry, ascending within a feature */
  const double* counts;        /* [nnz] counts, finite and > 0 */
  const double* sample_totals; /* [n] per-sample totals (table.cpp:55-62), > 0 */
} sf_problem;

/* Execution options. Zero-initialise for defaults. */
typedef struct sf_exec {
  int32_t n_devices;        /* devices to shard stripes over; 0 = all visible */
  const int32_t* devices;   /* explicit ordinals, or NULL for 0..n_devices-1 */
  int64_t mem_budget_bytes; /* per-device cap for embedding chunks; 0 = auto */
  int32_t kernel;           /* 0 = auto, 1 = dense tiled; unweighted only: 2 = sparse bit walk
                               (bitwise: the reference's adds in its order), 10 = split heavy
                               walk + light scatter (exact fixed-point sums, correctly rounded;
                               the default); weighted only: 11 = present-row walk (bitwise in
                               exact mode), 12 = u-walk, 13 = weighted split: dense heavy rows +
                               exact fixed-point light scatter (the default for WN / WU /
                               SF_GENERALIZED; falls back to 12 without the memory for it) */
  int32_t flags;            /* bit 0: SF_EXEC_EXACT_NO_FMA: bitwise-identical results (weighted:
                               no FMA; unweighted auto: the sparse walk instead of kernel 10) */
  double alpha;             /* SF_GENERALIZED only: the exponent, finite, >= 0 (ABI v3) */
} sf_exec;

#define SF_EXEC_EXACT_NO_FMA 1

/* Work and timing record of a run (all devices summed). */
typedef struct sf_stats {
  uint64_t updates_alg;  /* E * (stop-start) * n: the reference's unit of work */
  uint64_t updates_exec; /* node x slot updates the kernels actually executed */
  uint64_t launches;     /* kernel launches issued by the run */
  uint64_t n_chunks;     /* embedding chunks (postorder row ranges) */
  double embed_ms;       /* device time of the embedding kernels (max over devices) */
  double stripe_ms;      /* device time of the stripe kernels (max over devices) */
  double finalize_ms;    /* device time of finalize (max over devices) */
  double total_ms;       /* device time of the whole run (max over devices) */
  uint64_t fp64_ops;     /* FP64-pipe lane-ops of the DFMA heavy walk (kernel 10 with SF_HEAVY_GEMM=0),
                            the weighted u-walk (kernel 12) or the weighted split's dense heavy rows
                            (kernel 13: DADD + DFMA per heavy row and slot; fp32: the FP32 pipe); else 0 */
  uint64_t tensor_ops;   /* int8 tensor-core ops (2 per MAC) of the heavy-row GEMMs (kernel 10) */
  double tensor_ms;      /* device time of the heavy-row kernels: kernel 10's GEMMs, kernel 13's
                            dense kernel (sum of launches, max over devices) */
} sf_stats;

/* ---- library ------------------------------------------------------------ */
const char* sf_last_error(void);
const char* sf_version(void);
/* number of usable sm_100 devices (0 when none) */
int32_t sf_device_count(void);

/*
 * One-shot stripe computation: host problem in, host stripes out.
 * Replaces compute_unifrac<Real> (kernels.hpp:268-316): shear happened
 * before flattening; embedding, stripe update and (optionally) finalize run
 * on device; stop < 0 means total_stripes(n). tot_out may be NULL for
 * SF_WEIGHTED_UNNORMALIZED and must be non-NULL otherwise. With finalize,
 * dist_out holds d/t (0/0 -> 0) and tot_out the raw totals, exactly like a
 * finalized StripeSet. stats_out may be NULL.
 */
sf_status sf_compute_stripes(const sf_problem* p, sf_metric metric, sf_precision prec,
                             int32_t start, int32_t stop, void* dist_out, void* tot_out,
                             int32_t finalize, const sf_exec* ex, sf_stats* stats_out);

/* ---- plans: device-resident problem and stripes ------------------------ */
typedef struct sf_plan sf_plan;

/* Validate, upload the problem to each device and allocate its stripes. */
sf_status sf_plan_create(const sf_problem* p, sf_metric metric, sf_precision prec,
                         int32_t start, int32_t stop, const sf_exec* ex, sf_plan** out);
/* Zero the stripes, embed, accumulate every row, optionally finalize (async). */
sf_status sf_plan_run(sf_plan* plan, int32_t finalize);
/* Block until the plan's device work is done. */
sf_status sf_plan_sync(sf_plan* plan);
/* Copy stripes [start, stop) to host buffers (row-major, see above). */
sf_status sf_plan_download(sf_plan* plan, void* dist_out, void* tot_out);
/*
 * condense() (stripes.cpp:68-129) of a finalized full-range plan, on device:
 * out is the caller's row-major n x n fp64 matrix (zero diagonal, mirrored;
 * even n: the duplicated half-stripe copies must agree, else SF_EINVAL
 * "condense: duplicated slot disagrees"). The stripes never leave the GPU;
 * the matrix is copied to the host once.
 */
sf_status sf_plan_condense(sf_plan* plan, double* out);
/*
 * compute_distance_matrix<Real> (kernels.hpp:319-326): plan over [0, S),
 * run with finalize, sf_plan_condense into out (n x n). stats_out may be NULL.
 */
sf_status sf_compute_distance_matrix(const sf_problem* p, sf_metric metric, sf_precision prec, double* out,
                                     const sf_exec* ex, sf_stats* stats_out);
/*
 * Return the memory the library's per-device pool keeps for reuse across
 * plans to the device (the pool keeps freed plan buffers by default).
 */
sf_status sf_trim_memory(int32_t device);
/*
 * Write the plan's finalized stripes as a .strf file. Replaces
 * write_stripe_file (stripes.cpp:179-201): same 32-byte header, payload
 * (finalized distances, then raw totals for UW/WN) and FNV-1a checksum, so
 * read_stripe_file / merge of the reference read it. The stripes stream
 * from device memory through pinned staging (no full host copy). Refuses an
 * unfinalized plan like the reference; SF_GENERALIZED has no format code.
 */
sf_status sf_plan_write_strf(sf_plan* plan, const char* path);
sf_status sf_plan_stats(const sf_plan* plan, sf_stats* out);
void sf_plan_destroy(sf_plan* plan);

/*
 * Fold one host embedding batch into host stripe buffers. Replaces
 * accumulate() (kernels.hpp:232-248): emb is filled x padded row-major
 * (EmbeddingBatch::emb), lengths[filled]; dist/tot hold stripes
 * [start, stop) of an n-sample set and are updated in place. emb, lengths,
 * dist and tot share the precision `prec`.
 */
sf_status sf_accumulate_batch(const void* emb, const void* lengths, int32_t filled,
                              int32_t n_samples, int32_t padded, sf_metric metric,
                              sf_precision prec, int32_t start, int32_t stop,
                              void* dist_inout, void* tot_inout, int32_t device);

/*
 * Embedding rows [r0, r1) of the problem, built on device by the K1 kernels
 * and copied to `out` (row-major (r1-r0) x padded doubles, padding columns
 * zero). Replaces Embedder::next_batch (embed.cpp:42-82): weighted = summed
 * relative abundance, unweighted = 0/1 presence OR'ed up the tree.
 * `weighted` selects the mode (embed.hpp:30-34). Lengths are not returned
 * (they are the problem's lengths[r0..r1)).
 */
sf_status sf_embed_rows(const sf_problem* p, int32_t weighted, int32_t r0, int32_t r1,
                        double* out, int32_t padded, int32_t device);

/*
 * Divide distances by totals in place (0/0 -> 0) on device. Replaces
 * finalize() (kernels.hpp:251-259) for the ratio metrics; count = (stop-start)*n.
 */
sf_status sf_finalize(sf_precision prec, int64_t count, void* dist_inout, const void* tot,
                      int32_t device);

/*
 * Scatter finalized stripes [start, stop) of an n-sample matrix into the
 * n x n row-major double matrix `out` (caller-zeroed), mirroring condense()
 * (stripes.cpp:68-129). For even n, slots k >= n/2 of the last stripe are
 * verified against their first copy (exact for fp64, 1e-6 relative for fp32)
 * instead of written; a disagreement returns SF_EINVAL ("duplicated slot").
 * Call once per part, in increasing start order.
 */
sf_status sf_condense(sf_precision prec, int32_t n, int32_t start, int32_t stop,
                      const void* dist, double* out, int32_t device);

/*
 * Mantel permutation test on device. Replaces mantel (validate.cpp:111-159):
 * m1, m2 are n x n row-major distance matrices (DistanceMatrix::values);
 * r is the Pearson correlation of their condensed upper triangles and
 * p = (1 + #{r_perm >= r}) / (1 + permutations), permutation p relabelling
 * the samples of m2 with the reference's stream (mt19937_64 + std::shuffle
 * seeded from splitmix64(seed ^ splitmix64(p + 1))). Errors as the
 * reference: permutations < 1, n < 2, an asymmetric matrix (> 1e-12), zero
 * variance. r_squared is r * r. The sample-id check is the caller's.
 */
sf_status sf_mantel(int32_t n, const double* m1, const double* m2, int32_t permutations,
                    uint64_t seed, int32_t device, double* r_out, double* p_value_out);

/* Host-only: permutation p of the reference's Mantel stream (n entries). */
sf_status sf_mantel_permutation(int32_t n, uint64_t seed, int32_t p, int32_t* perm_out);

#ifdef __cplusplus
}
#endif

#endif /* STRIPEFRAC_CUDA_H_ */
