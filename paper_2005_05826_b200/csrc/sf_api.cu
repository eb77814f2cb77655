// C ABI of the B200 Striped-UniFrac hot path (include/stripefrac_cuda.h).
//
// Host side of compute_unifrac (kernels.hpp:268-316): validate, schedule the
// postorder embedding in row chunks, shard stripes over devices, launch
// K1 (embed) -> K2 (stripe update) per chunk, K3 (finalize), copy back.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <atomic>
#include <thread>
#include <string>
#include <vector>

#include "embed_kernels.cuh"
#include "gram_kernels.cuh"
#include "bits.cuh"
#include "split_kernels.cuh"
#include "sf_common.hpp"
#include "sparse_kernels.cuh"
#include "stripe_kernels.cuh"
#include "wsparse_kernels.cuh"
#include "wuwalk_kernels.cuh"
#include "wsplit_kernels.cuh"
#include "mantel_kernels.cuh"
#include "stripefrac_cuda.h"

namespace sf {

namespace {
thread_local std::string g_error;
}
void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

namespace {

#define SF_CUDA(expr)                                                                   \
  do {                                                                                  \
    const cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                            \
      set_error(std::string(#expr) + " failed: " + cudaGetErrorString(e_));             \
      return SF_ECUDA;                                                                  \
    }                                                                                   \
  } while (0)

#define SF_TRY(expr)                   \
  do {                                 \
    const sf_status st_ = (expr);      \
    if (st_ != SF_OK) return st_;      \
  } while (0)

sf_status fail(sf_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

// Device memory comes from a stream-ordered pool the library owns on each
// device (not the device's default pool, which torch / NCCL in the same
// process may use), with an unbounded release threshold: a plan's buffers
// (tens of GB at C3) go back to the pool when it is destroyed and the next
// plan takes them without new cudaMalloc/page-table work (plan creation was
// 70-300 ms of an end-to-end call; see tools/e2e_probe.py). sf_trim_memory()
// returns the pool's unused memory to the device.
struct PoolSlot {
  std::once_flag once;
  cudaMemPool_t pool = nullptr;
};
PoolSlot g_pools[64];

cudaMemPool_t device_pool(int device) {
  if (device < 0 || device >= 64) return nullptr;
  PoolSlot& s = g_pools[device];
  std::call_once(s.once, [&] {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      s.pool = pool;
    }
    cudaGetLastError();
  });
  return s.pool;
}

// Free device memory including what the library's pool holds but no buffer
// uses.
sf_status device_free_bytes(int device, size_t* out) {
  size_t freeb = 0, totalb = 0;
  SF_CUDA(cudaMemGetInfo(&freeb, &totalb));
  uint64_t reserved = 0, used = 0;
  cudaMemPool_t pool = device_pool(device);
  if (pool && cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
    freeb += static_cast<size_t>(reserved - used);
  cudaGetLastError();
  *out = freeb;
  return SF_OK;
}

// Test hook: SF_FORCE_PROBE_FAIL=1 makes every fit probe fail, so the
// free-memory fallback sizing runs.
bool probe_disabled() {
  const char* e = std::getenv("SF_FORCE_PROBE_FAIL");
  return e && std::atoi(e) != 0;
}

// Device allocation owned by one device.
struct DevBuf {
  int dev = -1;
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      int cur = -1;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaDeviceSynchronize();  // no kernel may still use it (the pool reuses it at once)
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
      if (cur >= 0) cudaSetDevice(cur);
    }
    p = nullptr;
    bytes = 0;
  }
  sf_status alloc(int device, size_t nbytes, const char* what) {
    reset();
    dev = device;
    if (nbytes == 0) nbytes = 16;
    cudaMemPool_t pool = device_pool(device);
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, nbytes, pool, 0) : cudaMallocAsync(&p, nbytes, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);  // usable from any stream
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return fail(SF_ENOMEM, std::string("cudaMalloc of ") + std::to_string(nbytes) +
                                 " bytes for " + what + " failed: " + cudaGetErrorString(e));
    }
    bytes = nbytes;
    return SF_OK;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Memory the library's pool holds for reuse (reserved, not in use).
size_t pool_free_bytes(int device) {
  uint64_t used = 0, reserved = 0;
  cudaMemPool_t pool = device_pool(device);
  if (!pool || cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) != cudaSuccess ||
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return reserved > used ? static_cast<size_t>(reserved - used) : 0;
}

// "Does `bytes` fit?" answered by a probe allocation from the library's
// pool (cudaMemGetInfo stalls up to ~100 ms on some calls: p99 63 ms on the
// box). The pool then keeps only `keep` of the probed bytes reserved (what
// the caller allocates next); the rest is trimmed back to the device.
bool probe_fits(int device, size_t bytes, size_t keep) {
  if (probe_disabled()) return false;
  bool ok = false;
  {
    DevBuf probe;
    ok = probe.alloc(device, bytes, "fit probe") == SF_OK;
  }
  cudaGetLastError();
  if (cudaMemPool_t pool = device_pool(device)) {
    uint64_t used = 0, reserved = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess)
      cudaMemPoolTrimTo(pool, static_cast<size_t>(used) + keep);
    if (std::getenv("SF_DEBUG") &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess)
      std::fprintf(stderr, "stripefrac: device %d pool: probe %zu MB %s, used %llu MB, reserved %llu MB\n", device,
                   bytes >> 20, ok ? "fits" : "fails", static_cast<unsigned long long>(used >> 20),
                   static_cast<unsigned long long>(reserved >> 20));
    cudaGetLastError();
  }
  return ok;
}

template <class T>
sf_status upload(DevBuf& b, int dev, const T* host, size_t count, cudaStream_t st,
                 const char* what) {
  SF_TRY(b.alloc(dev, count * sizeof(T), what));
  if (count) SF_CUDA(cudaMemcpyAsync(b.p, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return SF_OK;
}

int total_stripes(int n) { return n / 2; }

// ------------------------------------------------------------ devices
sf_status usable_devices(const sf_exec* ex, std::vector<int>& out) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(SF_ECUDA, "no CUDA device is available (this library has no CPU fallback)");
  }
  std::vector<int> want;
  if (ex && ex->devices && ex->n_devices > 0) {
    want.assign(ex->devices, ex->devices + ex->n_devices);
  } else {
    const int k = (ex && ex->n_devices > 0) ? std::min(ex->n_devices, count) : count;
    for (int i = 0; i < k; ++i) want.push_back(i);
  }
  // the architecture check is cached per ordinal: cudaGetDeviceProperties
  // measured 96-238 ms on some calls (tools/e2e_probe.py, SF_DEBUG), a
  // single attribute query is cheap, and the full properties are only
  // fetched for the error message
  static std::atomic<bool> checked[64] = {};
  for (int d : want) {
    if (d < 0 || d >= count) return fail(SF_EINVAL, "device ordinal " + std::to_string(d) + " out of range");
    if (d < 64 && checked[d].load(std::memory_order_relaxed)) continue;
    int major = 0;
    SF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d));
    if (major == 10) {
      if (d < 64) checked[d].store(true, std::memory_order_relaxed);
      continue;
    }
    cudaDeviceProp prop;
    SF_CUDA(cudaGetDeviceProperties(&prop, d));
    if (prop.major != 10)
      return fail(SF_ECUDA, std::string("device ") + std::to_string(d) + " (" + prop.name +
                                ") is not sm_100; this library is built for sm_100a only");
  }
  out = want;
  return SF_OK;
}

// ------------------------------------------------------------ validation
sf_status validate_table(const sf_problem* p);

// The tree part (rows, parents, lengths, leaf features) and the table part
// (CSR, counts, totals) of the problem; sf_plan_create starts the embedding
// schedule (which reads only the tree) between the two.
sf_status validate_problem(const sf_problem* p);
sf_status validate_tree(const sf_problem* p) {
  if (!p) return fail(SF_EINVAL, "problem is null");
  if (p->n_samples < 2)
    return fail(SF_EINVAL, "need at least 2 samples, got " + std::to_string(p->n_samples));
  if (p->n_rows < 1) return fail(SF_EINVAL, "embedding batch is empty");
  if (p->n_features < 1) return fail(SF_EINVAL, "table has no features");
  if (!p->parent_row || !p->lengths || !p->leaf_feature || !p->feat_ptr || !p->sample_idx ||
      !p->counts || !p->sample_totals)
    return fail(SF_EINVAL, "problem has a null array");
  const int E = p->n_rows;
  for (int r = 0; r < E; ++r) {
    const int par = p->parent_row[r];
    if (par != -1 && (par <= r || par >= E))
      return fail(SF_EINVAL, "row " + std::to_string(r) + " has an invalid parent row (rows must be in postorder)");
    const double L = p->lengths[r];
    if (!(L >= 0.0) || L > 1.7976931348623157e308)
      return fail(SF_EINVAL, "branch length must be finite and non-negative");
    const int f = p->leaf_feature[r];
    if (f < -1 || f >= p->n_features) return fail(SF_EINVAL, "leaf feature out of range");
  }
  std::vector<char> has_child(static_cast<size_t>(E), 0);
  for (int r = 0; r < E; ++r)
    if (p->parent_row[r] >= 0) has_child[static_cast<size_t>(p->parent_row[r])] = 1;
  for (int r = 0; r < E; ++r) {
    const bool leaf = p->leaf_feature[r] >= 0;
    if (leaf == static_cast<bool>(has_child[static_cast<size_t>(r)]))
      return fail(SF_EINVAL, "row " + std::to_string(r) +
                                 (leaf ? " is a leaf with children" : " is an internal row without children"));
  }
  return SF_OK;
}

sf_status validate_problem(const sf_problem* p) {
  SF_TRY(validate_tree(p));
  return validate_table(p);
}

sf_status validate_table(const sf_problem* p) {
  if (p->feat_ptr[0] != 0) return fail(SF_EINVAL, "feat_ptr[0] must be 0");
  for (int f = 0; f < p->n_features; ++f)
    if (p->feat_ptr[f + 1] < p->feat_ptr[f]) return fail(SF_EINVAL, "feat_ptr is not monotone");
  // the table entries (15M at C3) are checked by feature ranges on host
  // threads; the error reported is the first in feature order, as a
  // sequential scan would report it
  const int F = p->n_features;
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  std::vector<int> bad_f(static_cast<size_t>(T), F);
  std::vector<int> bad_kind(static_cast<size_t>(T), 0);
  auto scan = [&](int t) {
    const int f0 = static_cast<int>(static_cast<int64_t>(F) * t / T);
    const int f1 = static_cast<int>(static_cast<int64_t>(F) * (t + 1) / T);
    for (int f = f0; f < f1; ++f) {
      int prev = -1;
      for (int64_t e = p->feat_ptr[f]; e < p->feat_ptr[f + 1]; ++e) {
        const int smp = p->sample_idx[e];
        if (smp <= prev || smp >= p->n_samples) {
          bad_f[static_cast<size_t>(t)] = f;
          bad_kind[static_cast<size_t>(t)] = 1;
          return;
        }
        prev = smp;
        const double c = p->counts[e];
        if (!(c >= 0.0) || c > 1.7976931348623157e308) {
          bad_f[static_cast<size_t>(t)] = f;
          bad_kind[static_cast<size_t>(t)] = 2;
          return;
        }
      }
    }
  };
  if (p->feat_ptr[F] > (int64_t{1} << 20) && T > 1) {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(scan, t);
    for (auto& th : pool) th.join();
  } else {
    for (int t = 0; t < T; ++t) scan(t);
  }
  for (int t = 0; t < T; ++t) {  // lowest feature range first
    if (bad_kind[static_cast<size_t>(t)] == 1)
      return fail(SF_EINVAL, "sample indices of a feature must be ascending and in range");
    if (bad_kind[static_cast<size_t>(t)] == 2)
      return fail(SF_EINVAL, "count must be finite and non-negative");
  }
  for (int s = 0; s < p->n_samples; ++s)
    if (!(p->sample_totals[s] > 0.0))
      return fail(SF_EINVAL, "sample " + std::to_string(s) + " has no counts");
  return SF_OK;
}

sf_status validate_range(int n, int32_t start, int32_t& stop) {
  const int S = total_stripes(n);
  if (stop < 0) stop = S;
  if (start < 0 || stop > S || start >= stop)
    return fail(SF_EINVAL, "stripe range " + std::to_string(start) + ":" + std::to_string(stop) +
                               " does not fit in [0," + std::to_string(S) + ")");
  return SF_OK;
}

// ------------------------------------------------------------ schedule
struct Chunk {
  int32_t r0 = 0, r1 = 0;
  std::vector<int32_t> leaf_rows, leaf_feat;  // chunk-relative rows
  std::vector<int32_t> lvl_ptr;               // levels -> [int_rows)
  std::vector<int32_t> int_rows;              // chunk-relative internal rows
  std::vector<int32_t> cptr, codes;           // children location codes per int row
  std::vector<int32_t> carry_src, carry_dst;  // chunk rows -> pending slots
};

struct Schedule {
  std::vector<Chunk> chunks;
  int32_t n_pending = 0;
  int32_t cmax = 0;
};

// Single-chunk schedule (every row resident: the split, weighted-split and
// sparse walk paths): the same arrays as the general loop below, built with
// branch-free passes (leaf / internal rows interleave unpredictably in
// postorder), a counting sort by height and a threaded gather of the
// children codes.
Schedule build_schedule_single(const sf_problem* p) {
  const int E = p->n_rows;
  const int32_t* par = p->parent_row;
  const int32_t* lf = p->leaf_feature;
  std::vector<int32_t> height(static_cast<size_t>(E), 0), kptr(static_cast<size_t>(E) + 1, 0);
  int32_t nleaf = 0, hall = 0;
  for (int r = 0; r < E; ++r) {
    const int q = par[r];
    nleaf += lf[r] >= 0;
    if (q >= 0) {
      const int32_t h = height[static_cast<size_t>(r)] + 1;
      int32_t& hq = height[static_cast<size_t>(q)];
      hq = hq > h ? hq : h;
      hall = hall > h ? hall : h;
      ++kptr[static_cast<size_t>(q) + 1];
    }
  }
  for (int r = 0; r < E; ++r) kptr[static_cast<size_t>(r) + 1] += kptr[static_cast<size_t>(r)];
  std::vector<int32_t> kids(static_cast<size_t>(kptr[static_cast<size_t>(E)]));
  {
    std::vector<int32_t> at(kptr.begin(), kptr.end() - 1);
    for (int r = 0; r < E; ++r)  // ascending r: children in postorder = fold order
      if (par[r] >= 0) kids[static_cast<size_t>(at[static_cast<size_t>(par[r])]++)] = r;
  }
  Schedule sch;
  sch.cmax = E;
  sch.chunks.emplace_back();
  Chunk& c = sch.chunks.back();
  c.r0 = 0;
  c.r1 = E;
  c.leaf_rows.resize(static_cast<size_t>(nleaf) + 1);
  c.leaf_feat.resize(static_cast<size_t>(nleaf) + 1);
  int32_t hmax = 0;
  std::vector<int32_t> cnt(static_cast<size_t>(hall) + 2, 0);  // internal rows per height
  {
    int32_t j = 0;
    for (int r = 0; r < E; ++r) {  // branch-free compaction of the leaf rows
      const int32_t f = lf[r];
      c.leaf_rows[static_cast<size_t>(j)] = r;
      c.leaf_feat[static_cast<size_t>(j)] = f;
      j += f >= 0;
      const int32_t h = f >= 0 ? 0 : height[static_cast<size_t>(r)];
      hmax = hmax > h ? hmax : h;
      ++cnt[static_cast<size_t>(h) + 1];
    }
    c.leaf_rows.resize(static_cast<size_t>(nleaf));
    c.leaf_feat.resize(static_cast<size_t>(nleaf));
  }
  // internal rows by height, ascending rows within a height (stable)
  cnt[1] = 0;  // leaves (height 0) are not internal rows
  c.lvl_ptr.assign(1, 0);
  for (int h = 1; h <= hmax; ++h) {
    cnt[static_cast<size_t>(h) + 1] += cnt[static_cast<size_t>(h)];
    c.lvl_ptr.push_back(cnt[static_cast<size_t>(h) + 1]);
  }
  c.int_rows.resize(static_cast<size_t>(c.lvl_ptr.back()));
  for (int r = 0; r < E; ++r)
    if (lf[r] < 0) c.int_rows[static_cast<size_t>(cnt[static_cast<size_t>(height[static_cast<size_t>(r)])]++)] = r;
  // children codes in int_rows order (all chunk-relative: one chunk)
  const size_t NI = c.int_rows.size();
  c.cptr.resize(NI + 1);
  c.cptr[0] = 0;
  for (size_t i = 0; i < NI; ++i) {
    const int r = c.int_rows[i];
    c.cptr[i + 1] = c.cptr[i] + (kptr[static_cast<size_t>(r) + 1] - kptr[static_cast<size_t>(r)]);
  }
  c.codes.resize(static_cast<size_t>(c.cptr[NI]));
  auto gather = [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      const int r = c.int_rows[i];
      std::copy(kids.begin() + kptr[static_cast<size_t>(r)], kids.begin() + kptr[static_cast<size_t>(r) + 1],
                c.codes.begin() + c.cptr[i]);
    }
  };
  const unsigned T = NI > (1u << 16) ? std::max(1u, std::min(8u, std::thread::hardware_concurrency())) : 1u;
  if (T > 1) {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back(gather, NI * t / T, NI * (t + 1) / T);
    for (auto& th : pool) th.join();
  } else {
    gather(0, NI);
  }
  return sch;
}

// Postorder rows in chunks of <= cmax rows. Internal rows are grouped by
// height (children strictly lower), rows whose parent is in a later chunk
// are carried to pending slots, slots are recycled once consumed.
Schedule build_schedule(const sf_problem* p, int32_t cmax) {
  if (cmax >= p->n_rows) return build_schedule_single(p);
  const int E = p->n_rows;
  std::vector<int32_t> height(static_cast<size_t>(E), 0);
  std::vector<int32_t> kptr(static_cast<size_t>(E) + 1, 0), kids;
  for (int r = 0; r < E; ++r) {
    const int par = p->parent_row[r];
    if (par >= 0) {
      height[static_cast<size_t>(par)] = std::max(height[static_cast<size_t>(par)], height[static_cast<size_t>(r)] + 1);
      ++kptr[static_cast<size_t>(par) + 1];
    }
  }
  for (int r = 0; r < E; ++r) kptr[static_cast<size_t>(r) + 1] += kptr[static_cast<size_t>(r)];
  kids.assign(static_cast<size_t>(kptr[static_cast<size_t>(E)]), 0);
  {
    std::vector<int32_t> at(kptr.begin(), kptr.end() - 1);
    for (int r = 0; r < E; ++r)  // ascending r: children in postorder = fold order
      if (p->parent_row[r] >= 0) kids[static_cast<size_t>(at[static_cast<size_t>(p->parent_row[r])]++)] = r;
  }

  Schedule sch;
  sch.cmax = cmax;
  std::vector<int32_t> slot_of(static_cast<size_t>(E), -1);
  std::vector<int32_t> free_slots;
  for (int r0 = 0; r0 < E; r0 += cmax) {
    Chunk c;
    c.r0 = r0;
    c.r1 = std::min(E, r0 + cmax);
    c.leaf_rows.reserve(static_cast<size_t>(c.r1 - c.r0));
    c.leaf_feat.reserve(static_cast<size_t>(c.r1 - c.r0));
    c.codes.reserve(static_cast<size_t>(c.r1 - c.r0));
    c.cptr.reserve(static_cast<size_t>(c.r1 - c.r0) / 2 + 2);
    int32_t hmax = 0;
    for (int r = c.r0; r < c.r1; ++r) {
      if (p->leaf_feature[r] >= 0) {
        c.leaf_rows.push_back(r - c.r0);
        c.leaf_feat.push_back(p->leaf_feature[r]);
      } else {
        hmax = std::max(hmax, height[static_cast<size_t>(r)]);
      }
    }
    // bucket internal rows by height
    std::vector<int32_t> cnt(static_cast<size_t>(hmax) + 2, 0);
    for (int r = c.r0; r < c.r1; ++r)
      if (p->leaf_feature[r] < 0) ++cnt[static_cast<size_t>(height[static_cast<size_t>(r)]) + 1];
    c.lvl_ptr.push_back(0);
    for (int h = 1; h <= hmax; ++h) {
      cnt[static_cast<size_t>(h) + 1] += cnt[static_cast<size_t>(h)];
      c.lvl_ptr.push_back(cnt[static_cast<size_t>(h) + 1]);
    }
    c.int_rows.assign(static_cast<size_t>(c.lvl_ptr.back()), 0);
    std::vector<int32_t> at(cnt.begin() + 1, cnt.end());
    for (int r = c.r0; r < c.r1; ++r)
      if (p->leaf_feature[r] < 0) c.int_rows[static_cast<size_t>(at[static_cast<size_t>(height[static_cast<size_t>(r)]) - 1]++)] = r - c.r0;
    std::vector<int32_t> consumed;
    c.cptr.push_back(0);
    for (int32_t rel : c.int_rows) {
      const int r = c.r0 + rel;
      for (int32_t e = kptr[static_cast<size_t>(r)]; e < kptr[static_cast<size_t>(r) + 1]; ++e) {
        const int ch = kids[static_cast<size_t>(e)];
        if (ch >= c.r0) {
          c.codes.push_back(ch - c.r0);
        } else {
          c.codes.push_back(-1 - slot_of[static_cast<size_t>(ch)]);
          consumed.push_back(slot_of[static_cast<size_t>(ch)]);
        }
      }
      c.cptr.push_back(static_cast<int32_t>(c.codes.size()));
    }
    for (int32_t s : consumed) free_slots.push_back(s);
    for (int r = c.r0; r < c.r1; ++r) {
      const int par = p->parent_row[r];
      if (par >= c.r1) {
        int32_t slot;
        if (!free_slots.empty()) {
          slot = free_slots.back();
          free_slots.pop_back();
        } else {
          slot = sch.n_pending++;
        }
        slot_of[static_cast<size_t>(r)] = slot;
        c.carry_src.push_back(r - c.r0);
        c.carry_dst.push_back(slot);
      }
    }
    sch.chunks.push_back(std::move(c));
  }
  return sch;
}

// ------------------------------------------------------------ kernel table
using StripeFn = void (*)(const StripeArgs);

template <int M, class Real, int SRC, bool EXACT>
struct DenseCfg;
// fp64: 8 warps along samples (RK=8 each), 1 along stripes (RS=4) -> 64 x 128
template <int M, int SRC, bool EXACT>
struct DenseCfg<M, double, SRC, EXACT> {
  static constexpr int RK = 8, RS = 4, NWK = 8, NWS = 1, RB = 16;
};
template <int M, int SRC, bool EXACT>
struct DenseCfg<M, float, SRC, EXACT> {
  static constexpr int RK = 8, RS = 4, NWK = 8, NWS = 1, RB = 16;
};

template <int M, class Real, int SRC, bool EXACT>
void launch_dense(const StripeArgs& a, cudaStream_t st) {
  using C = DenseCfg<M, Real, SRC, EXACT>;
  constexpr int TK = C::NWK * C::RK;
  constexpr int TS = C::NWS * 32 * C::RS;
  const dim3 grid((a.n + TK - 1) / TK, (a.s_end - a.s_begin + TS - 1) / TS);
  stripe_dense_kernel<M, Real, SRC, EXACT, C::RK, C::RS, C::NWK, C::NWS, C::RB>
      <<<grid, 32 * C::NWK * C::NWS, 0, st>>>(a);
}

template <class Real, int SRC>
sf_status dispatch_dense(int metric, bool exact, const StripeArgs& a, cudaStream_t st) {
  switch (metric) {
    case SF_UNWEIGHTED:
      launch_dense<kUW, Real, SRC, false>(a, st);
      break;
    case SF_WEIGHTED_UNNORMALIZED:
      if (exact)
        launch_dense<kWU, Real, SRC, true>(a, st);
      else
        launch_dense<kWU, Real, SRC, false>(a, st);
      break;
    case SF_WEIGHTED_NORMALIZED:
      if (exact)
        launch_dense<kWN, Real, SRC, true>(a, st);
      else
        launch_dense<kWN, Real, SRC, false>(a, st);
      break;
    default:
      return fail(SF_EINVAL, "unknown metric");
  }
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

sf_status launch_stripes(int metric, int prec, int src, bool exact, const StripeArgs& a,
                         cudaStream_t st) {
  if (prec == SF_FP64) {
    if (src == kSrcBits) return dispatch_dense<double, kSrcBits>(metric, exact, a, st);
    if (src == kSrcF64) return dispatch_dense<double, kSrcF64>(metric, exact, a, st);
  } else {
    if (src == kSrcBits) return dispatch_dense<float, kSrcBits>(metric, exact, a, st);
    if (src == kSrcF64) return dispatch_dense<float, kSrcF64>(metric, exact, a, st);
    if (src == kSrcF32) return dispatch_dense<float, kSrcF32>(metric, exact, a, st);
  }
  return fail(SF_EINVAL, "unsupported precision/source combination");
}

int grid_for(int64_t count, int block) {
  int64_t g = (count + block - 1) / block;
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32));
}

}  // namespace
}  // namespace sf

using namespace sf;

// ------------------------------------------------------------ plan
struct DeviceState {
  int dev = -1;
  int32_t a = 0, b = 0;  // absolute stripe range on this device
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;     // D2H overlapped with the split kernel
  std::vector<cudaEvent_t> chunk_events;  // stripe chunks done (split kernel)
  // a finished block of the device's stripes: rows [row0, row0 + rows)
  // (relative to the device's first stripe) x columns [col0, col0 + cols)
  struct Span {
    int64_t row0, rows, col0, cols;
  };
  std::vector<Span> chunk_spans;  // one per chunk event
  bool defer_copy = false;  // record chunk events only; the caller stages the copies
  DevBuf lens, feat_ptr, sidx, counts, totals;
  DevBuf dist, tot, emb, pend, exec_ctr;
  DevBuf sched;  // all schedule arrays, packed
  std::vector<int64_t> sched_off;  // per chunk: offsets of its arrays in `sched`
  // sparse-bit (unweighted) path
  DevBuf nodebits, lens_pad;
  DevBuf cubtmp;  // scan scratch (weighted walks)
  size_t cub_bytes = 0;
  // split path (kernel 10): permuted rows, 64-row heavy words, limbs
  DevBuf limbs, fixbit, dmask, cacc, colsum;
  DevBuf fix, keys, vals, keys_out, perm, dense, sorttmp, nheavy;
  // light-row sums per slot, |S_e| per row; u-walk nonzero-word masks
  DevBuf lightsum, mcount, nzmask;
  DevBuf lcnt, lptr, lmem, lcur, lscantmp, lmem16;  // banded light scatter: member CSR + cursors of the light rows
  size_t lscan_bytes = 0;
  bool banded = false;
  // column-owned light scatter: entries (light rows containing each column)
  DevBuf ccnt, cptr, cent, cscantmp, linfo;
  size_t cscan_bytes = 0;
  bool light_columns = false;
  bool defer_light = false;  // column kernel launched per GEMM column group (tensor-core path)
  // deeper fixed-point levels: deep rows, their levels, member CSR, per-slot sums
  DevBuf drows, dfix, dcnt, dptr, dmem, dent, dcolsum, dcacc, deepsum, dscantmp;
  size_t dscan_bytes = 0;
  int64_t deep_entries = 0;
  // heavy rows on the tensor cores (gram_kernels.cuh): 0/1 rows B, digit
  // table, per-block digit planes A', GEMM output C, cuBLASLt state
  DevBuf gbits, growdig, gmask, gdj, gA, gC, gws;
  int64_t gram_kp = 0, gram_kpmax = 0;  // heavy rows (padded), digit-plane stride
  int64_t gram_h = 0;                   // heavy rows
  int32_t gram_nd = 0, gram_dj0 = 0;
  cublasLtHandle_t lt = nullptr;
  cublasLtMatmulDesc_t lt_op = nullptr;
  cublasLtMatrixLayout_t lt_a = nullptr, lt_b = nullptr, lt_c = nullptr;
  cublasLtMatmulAlgo_t lt_algo{};
  int64_t lt_m = 0, lt_n = 0, lt_k = 0;
  std::vector<cudaEvent_t> gemm_ev;  // (start, end) per heavy GEMM of the run
  size_t gemm_count = 0;
  uint64_t gemm_ops = 0;
  uint64_t heavy_updates = 0;  // (heavy row, slot) pairs the GEMMs covered (updates_exec)
  // weighted sparse walk (kernel 11): per chunk presence words, pool offsets, values
  DevBuf wnb, woff, wcnt, wpool;
  DevBuf wpoola, wA, wbase;  // kernel 12: generalized pool, column sums, pool base + chunk total
  // kernel 13: row counts / flags / scans, dense heavy rows, light member and
  // column lists, light column sums, the light part of every slot
  DevBuf ws_cnt, ws_hflag, ws_hidx, ws_lcnt, ws_lptr, ws_hmask, ws_lmask, ws_UH, ws_LH, ws_lmid, ws_lval,
      ws_ccnt, ws_cptr, ws_crow, ws_cval, ws_AL, ws_lightd, ws_tmp, ws_prank, ws_crank, ws_lvala, ws_lightt,
      ws_pool64;
  uint64_t host_fp64_ops = 0;  // FP64/FP32-pipe lane-ops counted on the host (kernel 13's dense part)
  DevBuf wnbo;               // kernel 12: combined (offset, presence word) cells
  int32_t light_pass = 0;  // stripes per light-sum pass (memory-bounded)
  // tensor-core path: the light sums are sized at run time, once the GEMM
  // operands (sized by the heavy-row count) are allocated
  bool light_lazy = false, light_sized = false;
  size_t sort_bytes = 0;
  std::vector<cudaEvent_t> events;
  uint64_t launches = 0;  // kernel launches of the last run on this device
  ~DeviceState() {
    if (dev >= 0) {
      cudaSetDevice(dev);
      if (stream) cudaStreamSynchronize(stream);
      if (copy_stream) cudaStreamSynchronize(copy_stream);
      for (auto e : events) cudaEventDestroy(e);
      for (auto e : chunk_events) cudaEventDestroy(e);
      for (auto e : gemm_ev) cudaEventDestroy(e);
      if (lt_a) cublasLtMatrixLayoutDestroy(lt_a);
      if (lt_b) cublasLtMatrixLayoutDestroy(lt_b);
      if (lt_c) cublasLtMatrixLayoutDestroy(lt_c);
      if (lt_op) cublasLtMatmulDescDestroy(lt_op);
      if (lt) cublasLtDestroy(lt);
      if (stream) cudaStreamDestroy(stream);
      if (copy_stream) cudaStreamDestroy(copy_stream);
    }
  }
};

struct sf_plan {
  int metric = 0, prec = 0;
  int32_t n = 0, E = 0, start = 0, stop = 0;
  bool bits = false, exact = false;
  // kernel 13: presence-bit embedding rows + a sparse value build (no dense
  // value rows); SF_WS_DENSE_EMBED=1 keeps the chunked dense build (A/B)
  bool wbits = false;
  size_t mem_budget = 0;  // sf_exec.mem_budget_bytes (0: none)
  double alpha = 1.0;  // generalized UniFrac exponent
  int kernel = 1;  // 1 dense, 2 sparse-bit walk, 10 split, 11 weighted present-row walk, 12 u-walk,
                   // 13 weighted split
  int32_t ws_G = 0, ws_nd = 8;  // kernel 13: fixed-point grid 2^-G of the light part, digit planes
  // split path: exact fixed-point levels of the lengths (fixed_levels)
  int32_t scale = 0, lo_bits = 32, vb = 63, levels = 1;
  std::vector<unsigned long long> fix, dfix;
  std::vector<int32_t> deep_rows;
  int64_t row_words = 0;  // per embedding row: words (bits) or doubles (values)
  Schedule sched;
  std::vector<std::unique_ptr<DeviceState>> devs;
  sf_stats stats{};
  bool ran = false;
  bool finalized = false;
};

namespace {

// Sparse node-packed bit kernel for the unweighted metric (kernel 2).
struct SparseCfg {
  static constexpr int RK = 4, RS = 2, NWK = 8, NWS = 2;
  static constexpr int TK = NWK * RK, TS = NWS * 32 * RS;
};

// Split (kernel 10): heavy rows walked warp-uniformly, light rows scattered.
// Weighted sparse walk (kernel 11).
struct WSparseCfg {
  static constexpr int RK = 4, RS = 2, NWK = 8, NWS = 2;
  static constexpr int TK = NWK * RK, TS = NWS * 32 * RS;
};

// Weighted u-walk (kernel 12).
struct WUWalkCfg {
  static constexpr int RS = 8, NW = 8;
};

#ifndef SF_SPLIT_V
#define SF_SPLIT_V 16
#endif
#ifndef SF_SPLIT_UC
#define SF_SPLIT_UC 1
#endif
#ifndef SF_SPLIT_NW
#define SF_SPLIT_NW 8
#endif
#ifndef SF_SPLIT_MINB
#define SF_SPLIT_MINB 2
#endif
#ifndef SF_SPLIT_FG
#define SF_SPLIT_FG 1
#endif
struct SplitCfg {
  static constexpr int V = SF_SPLIT_V, UC = SF_SPLIT_UC, NW = SF_SPLIT_NW, MINB = SF_SPLIT_MINB,
                       FG = SF_SPLIT_FG;
  static constexpr int RS = 16;  // light-band stripe height / download chunk unit: 512 stripes
  static constexpr int SCATTER_NW = 8;
};

// |X_e| threshold of the split path: rows at or above it are heavy (tensor-
// core GEMMs, cost ~ number of heavy rows), the rest light (scatter, cost ~
// pairs ~ |X_e|^2). Measured best with the column-owned light scatter:
// 0.04 at n = 25,000 (C3: 119.6 ms vs 122.0 at 0.03 and 123.1 at 0.05,
// profiles/r02_heavyfrac_c3_col3.jsonl); beyond, the size-aware form of
// round 1 (light pairs grow as x^2 and spread over more columns).
int split_heavy_min(int n) {
  // measured optima: 0.065 at C3 (profiles/r02_heavyfrac_c3_gemm_v4.jsonl,
  // the tensor-core path with the three-limb light kernel), 0.04 (25k/n)^(1/4)
  // at the C5 shard
  double frac = n > 25000 ? 0.04 * std::pow(25000.0 / n, 0.25) : 0.065;
  if (const char* e = std::getenv("SF_HEAVY_FRAC")) frac = std::atof(e);
  return std::max(2, static_cast<int>(frac * n));
}

int64_t sparse_n_ext(int n) {
  // a whole stripe tile past the last stripe: the widest is the split
  // kernel's 32 * RS (RS <= 16)
  // a whole tile past the last stripe: the DFMA walk's 32 V + UC columns, the
  // tensor-core path's GEMM block (<= 1024 u columns)
  const int64_t tile = std::max<int64_t>(std::max<int64_t>(SparseCfg::TK + SparseCfg::TS, 1024),
                                         std::max(32 * SplitCfg::RS, 32 * SplitCfg::V + SplitCfg::UC));
  const int64_t need = static_cast<int64_t>(n) + n / 2 + tile + 64;
  return (need + 3) / 4 * 4;
}

// Bytes the node-packed paths keep resident on one device (beyond stripes).
size_t nodepacked_bytes(int kernel, int32_t E, int n) {
  const int64_t W = (E + 31) / 32;
  const int64_t n_ext = sparse_n_ext(n);
  const size_t rows = static_cast<size_t>(E) * static_cast<size_t>((n + 31) / 32) * 4;
  if (kernel == 10) {  // + the light sums, (stripes x n) x 16 B, counted by the caller with stripes
    const int64_t W64 = (E + 63) / 64;
    return rows + static_cast<size_t>(W64 * n_ext) * 8 + static_cast<size_t>(W64) * 64 * 24 +
           static_cast<size_t>(E) * 32 + static_cast<size_t>(n) * 32;
  }
  return rows + static_cast<size_t>(W * n_ext) * 4 + static_cast<size_t>(W) * 32 * 8;
}

int ceil_log2(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

// Exact fixed-point levels of the branch lengths (split_kernels.cuh): every
// length L = sum_j v_j 2^-(scale + vb j) with integers v_j < 2^vb, by
// truncation from the top level down until the remainder is zero. Limb
// sums (hi = v >> lo_bits, lo) over up to E rows stay below 2^53, so they
// are exact in any order. A length on the main grid (every length within
// 2^(vb-53) of the longest, or with few significant bits) has one level.
struct FixedLevels {
  int32_t scale = 0, lo_bits = 32, vb = 63, levels = 1;
  std::vector<unsigned long long> fix;   // main level, [E]
  std::vector<int32_t> deep_rows;        // rows with a nonzero deeper level
  std::vector<unsigned long long> dfix;  // [deep row][levels - 1]
};

sf_status fixed_levels(const double* lengths, int32_t E, bool fp32, FixedLevels& out) {
  constexpr int kMaxLevels = 40;  // matches combine_levels (split_kernels.cuh)
  const int cl = ceil_log2(static_cast<int64_t>(E) + 1);
  out.lo_bits = std::min(32, 53 - cl);
  out.vb = std::min(63, out.lo_bits + (53 - cl));
  double lmax = 0.0;
  for (int32_t r = 0; r < E; ++r) {
    const double L = fp32 ? static_cast<double>(static_cast<float>(lengths[r])) : lengths[r];
    lmax = std::max(lmax, L);
  }
  out.scale = lmax > 0.0 ? out.vb - 1 - std::ilogb(lmax) : 0;
  out.fix.assign(static_cast<size_t>(E), 0ull);
  out.deep_rows.clear();
  out.dfix.clear();
  // main level from the double's bits (L = m 2^(x-1075), m < 2^53): v0 =
  // floor(m 2^(x-1075+scale)), the row is deep iff bits are shifted out;
  // rows split over host threads, deep rows (rare) take the exact ldexp
  // loop below, in row order
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  std::vector<std::vector<int32_t>> deep_of(static_cast<size_t>(T));
  auto main_level = [&](int t) {
    const int32_t r0 = static_cast<int32_t>(static_cast<int64_t>(E) * t / T);
    const int32_t r1 = static_cast<int32_t>(static_cast<int64_t>(E) * (t + 1) / T);
    for (int32_t r = r0; r < r1; ++r) {
      const double L = fp32 ? static_cast<double>(static_cast<float>(lengths[r])) : lengths[r];
      uint64_t bits;
      std::memcpy(&bits, &L, 8);
      const int x = static_cast<int>((bits >> 52) & 0x7ff);
      uint64_t m = bits & ((uint64_t{1} << 52) - 1);
      if (x) m |= uint64_t{1} << 52;
      const int sh = (x ? x - 1075 : -1074) + out.scale;
      uint64_t v = 0;
      bool deep = false;
      if (m == 0) {
        v = 0;
      } else if (sh >= 0) {
        v = m << sh;  // < 2^vb: L <= lmax
      } else if (sh > -64) {
        v = m >> -sh;
        deep = (m & ((uint64_t{1} << -sh) - 1)) != 0;
      } else {
        deep = true;
      }
      out.fix[static_cast<size_t>(r)] = v;
      if (deep) deep_of[static_cast<size_t>(t)].push_back(r);
    }
  };
  if (E > (1 << 16) && T > 1) {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(main_level, t);
    for (auto& th : pool) th.join();
  } else {
    for (int t = 0; t < T; ++t) main_level(t);
  }
  std::vector<std::vector<unsigned long long>> deep;  // per deep row, its levels 1..
  int levels = 1;
  for (const auto& rows : deep_of)
    for (int32_t r : rows) {
      double rem = fp32 ? static_cast<double>(static_cast<float>(lengths[r])) : lengths[r];
      // level j: v = floor(rem * 2^(scale + vb j)); rem -= v * 2^-(scale + vb j).
      // Both steps are exact: the scaled value and its floor are doubles, the
      // truncated part has no more significant bits than rem, and rem's low
      // bits are what the subtraction leaves.
      const double f0 = std::floor(std::ldexp(rem, out.scale));
      if (static_cast<unsigned long long>(f0) != out.fix[static_cast<size_t>(r)])
        return fail(SF_EINVAL, "fixed-point levels: main level mismatch (internal error)");
      rem -= std::ldexp(f0, -out.scale);
      std::vector<unsigned long long> v;
      for (int j = 1; rem != 0.0; ++j) {
        if (j >= kMaxLevels) return fail(SF_EINVAL, "branch lengths span too many binades for exact sums");
        const int sc = out.scale + out.vb * j;
        const double f = std::floor(std::ldexp(rem, sc));
        v.push_back(static_cast<unsigned long long>(f));
        rem -= std::ldexp(f, -sc);
      }
      levels = std::max(levels, 1 + static_cast<int>(v.size()));
      out.deep_rows.push_back(r);
      deep.push_back(std::move(v));
    }
  out.levels = levels;
  out.dfix.assign(deep.size() * static_cast<size_t>(levels - 1), 0ull);
  for (size_t i = 0; i < deep.size(); ++i)
    std::copy(deep[i].begin(), deep[i].end(), out.dfix.begin() + static_cast<int64_t>(i) * (levels - 1));
  return SF_OK;
}

// Split path (kernel 10): fixed-point levels on host, device arrays.
sf_status split_prepare(sf_plan* plan, DeviceState& d) {
  const int64_t E = plan->E;
  const int64_t W = (E + 63) / 64;
  const int64_t n_ext = sparse_n_ext(plan->n);
  SF_TRY(upload(d.fix, d.dev, plan->fix.data(), plan->fix.size(), d.stream, "fixed-point lengths"));
  SF_TRY(d.keys.alloc(d.dev, static_cast<size_t>(E) * 4, "row keys"));
  SF_TRY(d.keys_out.alloc(d.dev, static_cast<size_t>(E) * 4, "sorted keys"));
  SF_TRY(d.vals.alloc(d.dev, static_cast<size_t>(E) * 4, "row ids"));
  SF_TRY(d.perm.alloc(d.dev, static_cast<size_t>(E) * 4, "row permutation"));
  SF_TRY(d.dense.alloc(d.dev, static_cast<size_t>(E), "dense flags"));
  SF_TRY(d.nheavy.alloc(d.dev, 4, "heavy row count"));
  SF_TRY(d.dmask.alloc(d.dev, static_cast<size_t>(W) * 8, "dense-row mask"));
  SF_TRY(d.limbs.alloc(d.dev, static_cast<size_t>(W) * 64 * 16, "length limbs"));
  SF_TRY(d.fixbit.alloc(d.dev, static_cast<size_t>(W) * 64 * 8, "fixed-point lengths by bit"));
  SF_TRY(d.cacc.alloc(d.dev, 2 * sizeof(unsigned long long), "dense total"));
  SF_TRY(d.colsum.alloc(d.dev, static_cast<size_t>(plan->n) * 4 * sizeof(unsigned long long), "column sums"));
  SF_TRY(d.nodebits.alloc(d.dev, static_cast<size_t>(W * n_ext) * 8, "node-packed X words"));
  size_t stmp = 0;
  SF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, stmp, d.keys.as<uint32_t>(), d.keys_out.as<uint32_t>(),
                                          d.vals.as<int32_t>(), d.perm.as<int32_t>(), static_cast<int>(E),
                                          0, 1, d.stream));
  d.sort_bytes = stmp;
  SF_TRY(d.sorttmp.alloc(d.dev, stmp, "sort scratch"));
  const int R = static_cast<int>(plan->deep_rows.size());
  if (R > 0) {
    const int Jd = plan->levels - 1;
    SF_TRY(upload(d.drows, d.dev, plan->deep_rows.data(), plan->deep_rows.size(), d.stream, "deep rows"));
    SF_TRY(upload(d.dfix, d.dev, plan->dfix.data(), plan->dfix.size(), d.stream, "deep levels"));
    SF_TRY(d.dptr.alloc(d.dev, static_cast<size_t>(R + 1) * 4, "deep member offsets"));
    SF_TRY(d.dcnt.alloc(d.dev, static_cast<size_t>(R + 1) * 4, "deep member counts"));
    SF_TRY(d.dcolsum.alloc(d.dev, static_cast<size_t>(Jd) * plan->n * 4 * 8, "deep column sums"));
    SF_TRY(d.dcacc.alloc(d.dev, static_cast<size_t>(Jd) * 16, "deep dense totals"));
    size_t tmp = 0;
    SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d.dcnt.as<uint32_t>(), d.dptr.as<uint32_t>(), R + 1,
                                          d.stream));
    d.dscan_bytes = tmp;
    SF_TRY(d.dscantmp.alloc(d.dev, tmp, "deep scan scratch"));
  }
  return SF_OK;
}

// Light rows -> light sums of stripes [s0, s1) (lightsum row 0 = stripe s0);
// with_colsum: also add the light rows to the column sums (first pass only).
bool light_banded() {
  const char* e = std::getenv("SF_LIGHT_SCATTER");
  return !(e && std::atoi(e) == 0);
}

#ifndef SF_LIGHT_NT
#define SF_LIGHT_NT 1024
#endif
// Column-owned light scatter of stripes [p0, p1) for columns [k0, k1).
sf_status light_columns_run(sf_plan* plan, DeviceState& d, cudaStream_t st, int p0, int p1, int k0, int k1) {
  constexpr int NT = SF_LIGHT_NT;  // many warps: member-list reads and shared atomics in flight
  const int smem = 2 * kLightWin * 8;
  // test hook: SF_LIGHT_LIMB_MODE=1|2 forces the wider exact limb modes
  const int min_mode = std::getenv("SF_LIGHT_LIMB_MODE") ? std::atoi(std::getenv("SF_LIGHT_LIMB_MODE")) : 0;
  // entries per carry-folding chunk of the three-limb mode (<= 2048; test
  // hook SF_LIGHT_CHUNK_ENTRIES: tiny chunks fold carries often)
  int chunk = std::getenv("SF_LIGHT_CHUNK_ENTRIES") ? std::atoi(std::getenv("SF_LIGHT_CHUNK_ENTRIES")) : 2048;
  chunk = std::max(1, std::min(chunk, 2048));
  auto launch = [&](auto* kern, const auto* mem) -> sf_status {
    SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<std::max(1, std::min(k1 - k0, 65535)), NT, smem, st>>>(
        d.cptr.as<uint32_t>(), d.cent.as<uint2>(), d.linfo.as<LightRowInfo>(), mem, plan->lo_bits, plan->n, k0, k1,
        p0, p0, p1, d.lightsum.as<unsigned long long>(), d.exec_ctr.as<unsigned long long>(), min_mode, chunk);
    return SF_OK;
  };
  if (d.lmem16.p)
    SF_TRY(launch(sp_light_column_kernel<NT, uint16_t>, d.lmem16.as<uint16_t>()));
  else
    SF_TRY(launch(sp_light_column_kernel<NT, int32_t>, d.lmem.as<int32_t>()));
  SF_CUDA(cudaGetLastError());
  d.launches++;
  return SF_OK;
}

// Banded light scatter: member CSR once per run, then one launch per
// (512-stripe x KB-column) band of the pass, sized to stay in L2.
sf_status split_scatter_banded(sf_plan* plan, DeviceState& d, cudaStream_t st, int p0, int p1,
                               bool first) {
  const int n = plan->n;
  const int64_t E = plan->E;
  const int heavy_min = split_heavy_min(n);
  constexpr int NW = SplitCfg::SCATTER_NW;
  if (first) {
    sp_light_count_kernel<<<grid_for(E + 1, 256), 256, 0, st>>>(
        d.perm.as<int32_t>(), plan->E, n, d.nheavy.as<unsigned int>(), d.mcount.as<int32_t>(),
        d.lcnt.as<uint32_t>());
    size_t tmp = d.lscan_bytes;
    SF_CUDA(cub::DeviceScan::ExclusiveSum(d.lscantmp.p, tmp, d.lcnt.as<uint32_t>(), d.lptr.as<uint32_t>(),
                                          static_cast<int>(E + 1), st));
    const int blocks = static_cast<int>(std::min<int64_t>((E + NW - 1) / NW, 148 * 16));
    sp_light_members_kernel<<<blocks, 32 * NW, 0, st>>>(
        d.emb.as<uint32_t>(), plan->row_words, plan->E, n, d.perm.as<int32_t>(),
        d.nheavy.as<unsigned int>(), d.mcount.as<int32_t>(), d.lptr.as<uint32_t>(),
        d.fix.as<unsigned long long>(), plan->lo_bits, d.lmem.as<int32_t>(),
        d.colsum.as<unsigned long long>(), d.light_columns ? 2 : INT_MAX);
    SF_CUDA(cudaGetLastError());
    d.launches += 3;
  }
  if (d.light_columns) {
    if (first) {  // column-major entry CSR of the light member lists
      SF_CUDA(cudaMemsetAsync(d.ccnt.p, 0, static_cast<size_t>(n + 1) * 4, st));
      const int wblocks = static_cast<int>(std::min<int64_t>((E + 7) / 8, 148 * 16));
      sp_col_count_kernel<<<wblocks, 256, 0, st>>>(d.lmem.as<int32_t>(), d.lptr.as<uint32_t>(), plan->E,
                                                   d.nheavy.as<unsigned int>(), d.ccnt.as<uint32_t>());
      size_t tmp = d.cscan_bytes;
      SF_CUDA(cub::DeviceScan::ExclusiveSum(d.cscantmp.p, tmp, d.ccnt.as<uint32_t>(), d.cptr.as<uint32_t>(), n + 1,
                                            st));
      uint32_t M = 0, members = 0;
      SF_CUDA(cudaMemcpyAsync(&M, d.cptr.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
      SF_CUDA(cudaMemcpyAsync(&members, d.lptr.as<uint32_t>() + E, 4, cudaMemcpyDeviceToHost, st));
      SF_CUDA(cudaMemcpyAsync(d.ccnt.p, d.cptr.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToDevice, st));
      SF_CUDA(cudaStreamSynchronize(st));
      if (d.cent.bytes < static_cast<size_t>(M) * 8 + 8) SF_TRY(d.cent.alloc(d.dev, static_cast<size_t>(M) * 8 + 8, "column entries"));
      // 16-bit member lists for the column kernel (n <= 65536; SF_LIGHT_MEM16=0: 32-bit)
      const char* m16 = std::getenv("SF_LIGHT_MEM16");
      if (n <= 65536 && !(m16 && std::atoi(m16) == 0)) {
        if (d.lmem16.bytes < static_cast<size_t>(members) * 2 + 2)
          SF_TRY(d.lmem16.alloc(d.dev, static_cast<size_t>(members) * 2 + 2, "16-bit light members"));
        sp_narrow_members_kernel<<<grid_for(members, 256), 256, 0, st>>>(d.lmem.as<int32_t>(),
                                                                          d.lptr.as<uint32_t>() + E,
                                                                          d.lmem16.as<uint16_t>());
        d.launches++;
      } else {
        d.lmem16.reset();
      }
      sp_col_fill_kernel<<<wblocks, 256, 0, st>>>(d.lmem.as<int32_t>(), d.lptr.as<uint32_t>(), plan->E,
                                                  d.nheavy.as<unsigned int>(), d.ccnt.as<uint32_t>(),
                                                  d.cent.as<uint2>());
      // the light rows' column sums (rows with >= 2 members) from the entries
      sp_light_colsum_kernel<<<grid_for(static_cast<int64_t>(n) * 32, 256), 256, 0, st>>>(
          d.cptr.as<uint32_t>(), d.cent.as<uint2>(), d.perm.as<int32_t>(), d.mcount.as<int32_t>(),
          d.fix.as<unsigned long long>(), plan->lo_bits, n, d.colsum.as<unsigned long long>());
      d.launches++;
      if (d.linfo.bytes < static_cast<size_t>(E) * sizeof(LightRowInfo))
        SF_TRY(d.linfo.alloc(d.dev, static_cast<size_t>(E) * sizeof(LightRowInfo), "light row records"));
      sp_light_rowinfo_kernel<<<grid_for(E, 256), 256, 0, st>>>(d.perm.as<int32_t>(), plan->E,
                                                                 d.nheavy.as<unsigned int>(), d.lptr.as<uint32_t>(),
                                                                 d.fix.as<unsigned long long>(),
                                                                 d.linfo.as<LightRowInfo>());
      SF_CUDA(cudaGetLastError());
      d.launches += 4;
    }
    // the tensor-core path launches the column kernel per column group,
    // just before that group's GEMM blocks (light_columns_run)
    if (!d.defer_light) SF_TRY(light_columns_run(plan, d, st, p0, p1, 0, n));
    return SF_OK;
  }
  double band_mb = 32.0;  // measured: 32 MB <= 64 MB < 96 MB (profiles/r01_ab_c3_split_band*)
  if (const char* e = std::getenv("SF_LIGHT_BAND_MB")) band_mb = std::max(1e-3, std::atof(e));
  const int SB = 32 * SplitCfg::RS;
  const int64_t kb = static_cast<int64_t>(band_mb * 1048576.0 / (16.0 * SB));
  const int KB = static_cast<int>(std::max<int64_t>(std::min<int64_t>(256, n), std::min<int64_t>(kb, n)));
  const size_t smem = static_cast<size_t>(NW) * static_cast<size_t>(heavy_min) * 4;
  auto* kfirst = sp_light_band_kernel<NW, true>;
  auto* knext = sp_light_band_kernel<NW, false>;
  SF_CUDA(cudaFuncSetAttribute(kfirst, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  SF_CUDA(cudaFuncSetAttribute(knext, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = static_cast<int>(std::min<int64_t>((E + NW - 1) / NW, 148 * 16));
  for (int s0 = p0; s0 < p1; s0 += SB) {
    const int s1 = std::min(p1, s0 + SB);
    for (int k0 = 0; k0 < n; k0 += KB) {
      auto* kern = s0 == p0 ? kfirst : knext;  // first band of the pass: search, store cursors
      kern<<<blocks, 32 * NW, smem, st>>>(d.perm.as<int32_t>(), plan->E, n, d.nheavy.as<unsigned int>(),
                                          d.lptr.as<uint32_t>(), d.lmem.as<int32_t>(), d.lcur.as<uint16_t>(),
                                          d.fix.as<unsigned long long>(), plan->lo_bits, p0, s0, s1, k0,
                                          std::min(n, k0 + KB), d.lightsum.as<unsigned long long>(),
                                          d.exec_ctr.as<unsigned long long>(), heavy_min);
      d.launches++;
    }
  }
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

// Deeper fixed-point levels: member lists of the deep rows (first pass) and
// their pair sums for stripes [s0, s1) into d.deepsum.
sf_status split_scatter_deep(sf_plan* plan, DeviceState& d, cudaStream_t st, int s0, int s1, bool first) {
  const int R = static_cast<int>(plan->deep_rows.size());
  if (R == 0) return SF_OK;
  const int n = plan->n;
  const int J = plan->levels;
  if (first) {
    SF_CUDA(cudaMemsetAsync(d.dcolsum.p, 0, d.dcolsum.bytes, st));
    SF_CUDA(cudaMemsetAsync(d.dcacc.p, 0, d.dcacc.bytes, st));
    sp_deep_count_kernel<<<grid_for(R + 1, 256), 256, 0, st>>>(d.drows.as<int32_t>(), R, n, d.mcount.as<int32_t>(),
                                                                 d.dcnt.as<uint32_t>());
    size_t tmp = d.dscan_bytes;
    SF_CUDA(cub::DeviceScan::ExclusiveSum(d.dscantmp.p, tmp, d.dcnt.as<uint32_t>(), d.dptr.as<uint32_t>(), R + 1,
                                          st));
    uint32_t M = 0;
    SF_CUDA(cudaMemcpyAsync(&M, d.dptr.as<uint32_t>() + R, 4, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
    d.deep_entries = M;
    if (d.dmem.bytes < static_cast<size_t>(M) * 4 + 4) {
      SF_TRY(d.dmem.alloc(d.dev, static_cast<size_t>(M) * 4 + 4, "deep members"));
      SF_TRY(d.dent.alloc(d.dev, static_cast<size_t>(M) * 4 + 4, "deep member rows"));
    }
    sp_deep_members_kernel<<<grid_for(static_cast<int64_t>(R) * 32, 256), 256, 0, st>>>(
        d.emb.as<uint32_t>(), plan->row_words, n, d.drows.as<int32_t>(), R, d.mcount.as<int32_t>(),
        d.dptr.as<uint32_t>(), d.dfix.as<unsigned long long>(), J, plan->lo_bits, d.dmem.as<int32_t>(),
        d.dent.as<uint32_t>(), d.dcolsum.as<unsigned long long>(), d.dcacc.as<unsigned long long>());
    SF_CUDA(cudaGetLastError());
    d.launches += 3;
  }
  if (d.deep_entries > 0) {
    sp_deep_scatter_kernel<<<grid_for(d.deep_entries * 32, 256), 256, 0, st>>>(
        d.dptr.as<uint32_t>(), d.dmem.as<int32_t>(), d.dent.as<uint32_t>(), d.deep_entries,
        d.dfix.as<unsigned long long>(), J, plan->lo_bits, n, s0, s1, d.deepsum.as<unsigned long long>());
    SF_CUDA(cudaGetLastError());
    d.launches++;
  }
  return SF_OK;
}

// Light-sum passes: the whole stripe range if its light sums (and deeper
// levels' pair sums) fit next to everything else plus `after` bytes still to
// be allocated, else passes of whole 512-stripe tiles; allocates them.
sf_status light_sums_alloc(sf_plan* plan, DeviceState& d, size_t after) {
  const int n = plan->n;
  size_t freeb = 0;
  // light sums (hi, lo) and the deeper levels' pair sums per slot
  const size_t per_stripe = static_cast<size_t>(n) * 16 * static_cast<size_t>(plan->levels);
  const size_t reserve = (1ull << 30);
  const int span = d.b - d.a;
  // without a budget, a probe allocation of the whole range plus `after` and
  // the reserve answers "does it fit"; it returns to the pool for the
  // allocations below. cudaMemGetInfo stalls up to ~100 ms on some calls
  // (p99 63 ms on the box).
  size_t fit = 0;
  bool probed = false;
  if (plan->mem_budget == 0 && !std::getenv("SF_LIGHT_PASS")) {
    const size_t need = static_cast<size_t>(span) * per_stripe + after;
    // steady state: the pool still holds the previous plan's freed blocks,
    // so the same allocations are served again without a probe (a probe's
    // single large block would fragment them)
    // (the reserve is headroom for allocations outside the pool: in the
    // steady state they exist already, so free pool bytes >= need suffice)
    if (pool_free_bytes(d.dev) >= need || probe_fits(d.dev, need + reserve, need)) {
      fit = static_cast<size_t>(span);
      probed = true;
    }
  }
  if (!probed) {
    SF_TRY(device_free_bytes(d.dev, &freeb));
    fit = freeb > reserve + after ? (freeb - reserve - after) / per_stripe : 0;
  }
  if (plan->mem_budget > 0) fit = std::min(fit, plan->mem_budget / per_stripe);
  int pass = static_cast<int>(std::min<size_t>(fit, static_cast<size_t>(span)));
  if (pass < span) pass = std::max(512, pass / 512 * 512);
  if (const char* e = std::getenv("SF_LIGHT_PASS")) pass = std::max(1, std::atoi(e));  // tests
  d.light_pass = std::min(pass, span);
  if (std::getenv("SF_DEBUG"))
    std::fprintf(stderr, "stripefrac: device %d stripes [%d,%d): light pass %d stripes (%s)\n", d.dev, d.a, d.b,
                 d.light_pass, probed ? "probe fit" : ("free " + std::to_string(freeb >> 20) + " MB").c_str());
  SF_TRY(d.lightsum.alloc(d.dev, static_cast<size_t>(d.light_pass) * n * 16, "light-row sums"));
  if (plan->levels > 1)
    SF_TRY(d.deepsum.alloc(d.dev, static_cast<size_t>(d.light_pass) * n * 16 * (plan->levels - 1),
                           "deep-level sums"));
  return SF_OK;
}

sf_status split_scatter(sf_plan* plan, DeviceState& d, cudaStream_t st, int s0, int s1, bool with_colsum) {
  const int n = plan->n;
  const int64_t E = plan->E;
  const int heavy_min = split_heavy_min(n);
  const size_t cells = static_cast<size_t>(s1 - s0) * static_cast<size_t>(n);
  // the column-owned scatter writes every light-sum cell of the pass
  if (!(d.banded && d.light_columns)) SF_CUDA(cudaMemsetAsync(d.lightsum.p, 0, cells * 16, st));
  if (plan->levels > 1) SF_CUDA(cudaMemsetAsync(d.deepsum.p, 0, cells * 16 * (plan->levels - 1), st));
  SF_TRY(split_scatter_deep(plan, d, st, s0, s1, with_colsum));
  if (d.banded) return split_scatter_banded(plan, d, st, s0, s1, with_colsum);
  constexpr int NW = SplitCfg::SCATTER_NW;
  const size_t smem = static_cast<size_t>(NW) * static_cast<size_t>(heavy_min) * 4;
  auto* kern = sp_light_scatter_kernel<NW, 8>;
  SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = static_cast<int>(std::min<int64_t>((E + NW - 1) / NW, 148 * 16));
  kern<<<blocks, 32 * NW, smem, st>>>(d.emb.as<uint32_t>(), plan->row_words, plan->E, n, d.perm.as<int32_t>(),
                                     d.nheavy.as<unsigned int>(), d.mcount.as<int32_t>(),
                                     d.fix.as<unsigned long long>(), plan->lo_bits, s0, s1,
                                     d.lightsum.as<unsigned long long>(),
                                     with_colsum ? d.colsum.as<unsigned long long>() : nullptr,
                                     d.exec_ctr.as<unsigned long long>(), heavy_min);
  SF_CUDA(cudaGetLastError());
  d.launches++;
  return SF_OK;
}

sf_status split_build(sf_plan* plan, DeviceState& d, cudaStream_t st) {
  const int n = plan->n;
  const int64_t E = plan->E;
  const int64_t W = (E + 63) / 64;
  const int64_t n_ext = sparse_n_ext(n);
  const int64_t stride = plan->row_words;
  const int heavy_min = split_heavy_min(n);
  SF_CUDA(cudaMemsetAsync(d.dmask.p, 0, static_cast<size_t>(W) * 8, st));
  SF_CUDA(cudaMemsetAsync(d.cacc.p, 0, 2 * sizeof(unsigned long long), st));
  SF_CUDA(cudaMemsetAsync(d.colsum.p, 0, static_cast<size_t>(n) * 4 * sizeof(unsigned long long), st));
  SF_CUDA(cudaMemsetAsync(d.nheavy.p, 0, 4, st));
  sp_row_key_kernel<<<grid_for(E * 32, 256), 256, 0, st>>>(
      d.emb.as<uint32_t>(), stride, plan->E, n, heavy_min, d.keys.as<uint32_t>(), d.vals.as<int32_t>(),
      d.dense.as<uint8_t>(), d.nheavy.as<unsigned int>(), d.mcount.as<int32_t>());
  size_t stmp = d.sort_bytes;
  SF_CUDA(cub::DeviceRadixSort::SortPairs(d.sorttmp.p, stmp, d.keys.as<uint32_t>(), d.keys_out.as<uint32_t>(),
                                          d.vals.as<int32_t>(), d.perm.as<int32_t>(), static_cast<int>(E),
                                          0, 1, st));
  sp_perm_kernel<<<grid_for(W * 64, 256), 256, 0, st>>>(
      d.perm.as<int32_t>(), plan->E, W * 64, d.dense.as<uint8_t>(), d.fix.as<unsigned long long>(),
      plan->lo_bits, d.dmask.as<unsigned long long>(), d.limbs.as<double2>(), d.fixbit.as<unsigned long long>(),
      d.cacc.as<unsigned long long>());
  sp_transpose_kernel<<<grid_for(W * stride * 32, 256), 256, 0, st>>>(
      d.emb.as<uint32_t>(), stride, d.perm.as<int32_t>(), d.nheavy.as<unsigned int>(), n,
      d.dmask.as<unsigned long long>(), d.nodebits.as<unsigned long long>(), n_ext);
  sp_extend_kernel<<<grid_for(W * (n_ext - n), 256), 256, 0, st>>>(
      d.nodebits.as<unsigned long long>(), n_ext, n, d.nheavy.as<unsigned int>());
  sp_heavy_colsum_kernel<<<grid_for(static_cast<int64_t>(kHeavyColSlices) * n, 256), 256, 0, st>>>(
      d.nodebits.as<unsigned long long>(), n_ext, n, d.nheavy.as<unsigned int>(),
      d.dmask.as<unsigned long long>(), d.fixbit.as<unsigned long long>(), plan->lo_bits,
      d.colsum.as<unsigned long long>());
  SF_CUDA(cudaGetLastError());
  d.launches += 7;  // key, sort, perm, transpose, extend, colsum (+ memsets)
  // first light pass (the one that also adds the light rows' column sums)
  // tensor-core path with run-time light sums: the member lists and the
  // column CSR now; the first pass's deep scatter once the sums exist
  if (d.light_lazy) return split_scatter_banded(plan, d, st, d.a, std::min(d.b, d.a + d.light_pass), true);
  return split_scatter(plan, d, st, d.a, std::min(d.b, d.a + d.light_pass), true);
}

// Heavy-walk tile (SplitCfg): V v-slots per lane x UC u columns per warp,
// NW warps per CTA, MINB CTAs per SM (register cap), FG factors formed
// ahead of their DFMAs. The tile shape is a compile-time choice
// (-DSF_SPLIT_V=... etc. builds the A/B libraries of tools/build_ab.sh).
template <class Real>
sf_status launch_split(const SplitArgs& a, cudaStream_t st) {
  constexpr int V = SplitCfg::V, UC = SplitCfg::UC, NW = SplitCfg::NW;
  const int64_t cols = (static_cast<int64_t>(a.n) + UC - 1) / UC;
  const dim3 grid(static_cast<unsigned>((cols + NW - 1) / NW),
                  static_cast<unsigned>((a.s_end - a.s_begin + UC - 1 + 32 * V - 1) / (32 * V)));
  stripe_split_kernel<Real, V, UC, NW, SplitCfg::MINB, SplitCfg::FG><<<grid, 32 * NW, 0, st>>>(a);
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

// ---- heavy rows on the tensor cores (gram_kernels.cuh) ----------------------
#define SF_LT(expr)                                                                       \
  do {                                                                                    \
    const cublasStatus_t s_ = (expr);                                                     \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                      \
      return fail(SF_ECUDA, std::string(#expr) + " failed: cuBLASLt status " + std::to_string(static_cast<int>(s_))); \
  } while (0)

// The tensor-core heavy path is the default; SF_HEAVY_GEMM=0 selects the
// DFMA heavy walk (stripe_split_kernel) for A/B and the bitwise cross-check.
bool heavy_gemm_enabled() {
  const char* e = std::getenv("SF_HEAVY_GEMM");
  return !(e && std::atoi(e) == 0);
}

// u columns per GEMM block: the window of v columns a block reads is
// (stripes + BK - 1) wide, so smaller blocks waste less on short stripe
// ranges; 1024 at the full C3 range.
int gram_block(int span) {
  if (const char* e = std::getenv("SF_GRAM_BK")) return std::max(16, std::atoi(e) / 16 * 16);
  int bk = 1024;
  while (bk > 128 && span < 4 * bk) bk /= 2;
  return bk;
}

// Once per run, after split_build: heavy-row count and digit planes to host,
// the 0/1 rows B (all n_ext columns) and the digit table.
sf_status gram_prepare(sf_plan* plan, DeviceState& d, cudaStream_t st) {
  const int64_t n_ext = sparse_n_ext(plan->n);
  const int64_t W64 = (static_cast<int64_t>(plan->E) + 63) / 64;
  if (d.gmask.bytes < 8) SF_TRY(d.gmask.alloc(d.dev, 8, "digit plane mask"));
  SF_CUDA(cudaMemsetAsync(d.gmask.p, 0, 8, st));
  // digits of every permuted row (a bound on the heavy rows: all rows)
  const int64_t kp_max = (W64 * 64 + 127) / 128 * 128;
  d.gram_kpmax = kp_max;
  if (d.growdig.bytes < static_cast<size_t>(kp_max) * kMaxDigits)
    SF_TRY(d.growdig.alloc(d.dev, static_cast<size_t>(kp_max) * kMaxDigits, "row digits"));
  sp_gram_rowdig_kernel<<<grid_for(kp_max, 256), 256, 0, st>>>(d.fixbit.as<unsigned long long>(),
                                                                 d.nheavy.as<unsigned int>(), kp_max,
                                                                 d.growdig.as<int8_t>(), d.gmask.as<unsigned int>());
  SF_CUDA(cudaGetLastError());
  unsigned int hm[2] = {0u, 0u};
  SF_CUDA(cudaMemcpyAsync(hm, d.nheavy.p, 4, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaMemcpyAsync(hm + 1, d.gmask.p, 4, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  const int64_t H = hm[0];
  const int64_t Kp = std::max<int64_t>(128, (H + 127) / 128 * 128);
  std::vector<int32_t> dj;
  for (int j = 0; j < kMaxDigits; ++j)
    if (hm[1] & (1u << j)) dj.push_back(j);
  if (dj.empty()) dj.push_back(0);  // no heavy length: one (zero) plane keeps the shapes valid
  d.gram_kp = Kp;
  d.gram_h = H;
  d.gram_nd = static_cast<int32_t>(dj.size());
  d.gram_dj0 = dj.front();
  for (size_t j = 1; j < dj.size(); ++j)
    if (dj[j] != dj[j - 1] + 1) d.gram_dj0 = -1;
  if (d.gdj.bytes < dj.size() * 4) SF_TRY(d.gdj.alloc(d.dev, kMaxDigits * 4, "digit planes"));
  SF_CUDA(cudaMemcpyAsync(d.gdj.p, dj.data(), dj.size() * 4, cudaMemcpyHostToDevice, st));
  const size_t bbytes = static_cast<size_t>(n_ext) * static_cast<size_t>(Kp);
  if (d.gbits.bytes < bbytes) SF_TRY(d.gbits.alloc(d.dev, bbytes, "heavy 0/1 rows"));
  sp_gram_bits_kernel<<<grid_for((Kp / 64) * n_ext, 256), 256, 0, st>>>(
      d.nodebits.as<unsigned long long>(), n_ext, d.nheavy.as<unsigned int>(), Kp, d.gbits.as<int8_t>());
  SF_CUDA(cudaGetLastError());
  d.launches += 2;
  return SF_OK;
}

// cuBLASLt int8 GEMM C (M x N, int32, col-major) = A^T B, A stored K x M and
// B stored K x N (both K-contiguous), shapes cached per device.
sf_status gram_matmul(DeviceState& d, int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* B, int32_t* C,
                      cudaStream_t st) {
  if (!d.lt) SF_LT(cublasLtCreate(&d.lt));
  if (!d.lt_op) {
    SF_LT(cublasLtMatmulDescCreate(&d.lt_op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    SF_LT(cublasLtMatmulDescSetAttribute(d.lt_op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    SF_LT(cublasLtMatmulDescSetAttribute(d.lt_op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
  }
  constexpr size_t kWorkspace = size_t{64} << 20;
  if (d.gws.bytes < kWorkspace) SF_TRY(d.gws.alloc(d.dev, kWorkspace, "GEMM workspace"));
  if (M != d.lt_m || N != d.lt_n || K != d.lt_k) {
    if (d.lt_a) cublasLtMatrixLayoutDestroy(d.lt_a);
    if (d.lt_b) cublasLtMatrixLayoutDestroy(d.lt_b);
    if (d.lt_c) cublasLtMatrixLayoutDestroy(d.lt_c);
    d.lt_a = d.lt_b = d.lt_c = nullptr;
    d.lt_m = d.lt_n = d.lt_k = 0;
    SF_LT(cublasLtMatrixLayoutCreate(&d.lt_a, CUDA_R_8I, static_cast<uint64_t>(K), static_cast<uint64_t>(M), K));
    SF_LT(cublasLtMatrixLayoutCreate(&d.lt_b, CUDA_R_8I, static_cast<uint64_t>(K), static_cast<uint64_t>(N), K));
    SF_LT(cublasLtMatrixLayoutCreate(&d.lt_c, CUDA_R_32I, static_cast<uint64_t>(M), static_cast<uint64_t>(N), M));
    cublasLtMatmulPreference_t pref = nullptr;
    SF_LT(cublasLtMatmulPreferenceCreate(&pref));
    struct PrefGuard {
      cublasLtMatmulPreference_t p;
      ~PrefGuard() { cublasLtMatmulPreferenceDestroy(p); }
    } pg{pref};
    const size_t ws = kWorkspace;
    SF_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws)));
    // the chosen algorithm per (device, shape) is cached process-wide: every
    // plan of the same problem asks for the same shapes
    static std::mutex mu;
    static std::vector<std::pair<std::array<int64_t, 4>, cublasLtMatmulAlgo_t>> cache;
    const std::array<int64_t, 4> key{d.dev, M, N, K};
    bool hit = false;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (const auto& c : cache)
        if (c.first == key) {
          d.lt_algo = c.second;
          hit = true;
        }
    }
    if (!hit) {
      cublasLtMatmulHeuristicResult_t res{};
      int nres = 0;
      SF_LT(cublasLtMatmulAlgoGetHeuristic(d.lt, d.lt_op, d.lt_a, d.lt_b, d.lt_c, d.lt_c, pref, 1, &res, &nres));
      if (nres < 1) return fail(SF_ECUDA, "cuBLASLt has no int8 GEMM for this shape");
      d.lt_algo = res.algo;
      std::lock_guard<std::mutex> lk(mu);
      cache.emplace_back(key, res.algo);
    }
    d.lt_m = M, d.lt_n = N, d.lt_k = K;
  }
  const int32_t alpha = 1, beta = 0;
  SF_LT(cublasLtMatmul(d.lt, d.lt_op, &alpha, A, d.lt_a, B, d.lt_b, &beta, C, d.lt_c, C, d.lt_c, &d.lt_algo,
                       d.gws.p, kWorkspace, st));
  return SF_OK;
}

// Stripes [c0, c1) of the plan's device: per block of BK u columns, its
// digit planes, one GEMM against the window of v columns, the epilogue.
sf_status gram_run(sf_plan* plan, DeviceState& d, int c0, int c1, int gl_begin, int32_t finalize,
                   cudaStream_t st, int k_begin, int k_end) {
  const int n = plan->n;
  const int span = c1 - c0;
  const int bk = gram_block(span);
  const int64_t Kp = d.gram_kp;
  const int nd = d.gram_nd;
  const int64_t M = static_cast<int64_t>(bk) * nd;
  const int64_t W = span + bk - 1;  // window columns
  if (d.gA.bytes < static_cast<size_t>(M * Kp)) SF_TRY(d.gA.alloc(d.dev, static_cast<size_t>(M * Kp), "digit planes A"));
  if (d.gC.bytes < static_cast<size_t>(M * W) * 4) SF_TRY(d.gC.alloc(d.dev, static_cast<size_t>(M * W) * 4, "GEMM output"));
  GramArgs g;
  g.C = d.gC.as<int32_t>();
  g.dj = d.gdj.as<int32_t>();
  g.dj0 = d.gram_dj0;
  g.nd = nd;
  g.bk = bk;
  g.c0 = c0;
  g.c1 = c1;
  g.M = M;
  g.n = n;
  g.out_begin = d.a;
  g.gl_begin = gl_begin;
  g.lo_bits = plan->lo_bits;
  g.scale = plan->scale;
  g.finalize = finalize ? 1 : 0;
  g.levels = plan->levels;
  g.vb = plan->vb;
  g.dacc = plan->levels > 1 ? d.deepsum.as<unsigned long long>() : nullptr;
  g.dcolsum = plan->levels > 1 ? d.dcolsum.as<unsigned long long>() : nullptr;
  g.dcacc = plan->levels > 1 ? d.dcacc.as<unsigned long long>() : nullptr;
  g.gl = d.lightsum.as<unsigned long long>();
  g.colsum = d.colsum.as<unsigned long long>();
  g.cacc = d.cacc.as<unsigned long long>();
  g.dist = d.dist.p;
  g.tot = d.tot.p;
  for (int k0 = k_begin; k0 < k_end; k0 += bk) {
    sp_gram_digits_kernel<<<grid_for(static_cast<int64_t>(bk) * (Kp / 16), 256), 256, 0, st>>>(
        d.gbits.as<int8_t>(), Kp, k0, bk, n, d.growdig.as<int8_t>(), d.gram_kpmax, d.gdj.as<int32_t>(), nd,
        d.gA.as<int8_t>());
    SF_CUDA(cudaGetLastError());
    const int64_t l_start = static_cast<int64_t>(k0) + c0 + 1;  // < n_ext - W (sparse_n_ext)
    while (d.gemm_ev.size() < 2 * (d.gemm_count + 1)) {
      cudaEvent_t e;
      SF_CUDA(cudaEventCreate(&e));
      d.gemm_ev.push_back(e);
    }
    SF_CUDA(cudaEventRecord(d.gemm_ev[2 * d.gemm_count], st));
    SF_TRY(gram_matmul(d, M, W, Kp, d.gA.as<int8_t>(), d.gbits.as<int8_t>() + l_start * Kp, d.gC.as<int32_t>(), st));
    SF_CUDA(cudaEventRecord(d.gemm_ev[2 * d.gemm_count + 1], st));
    ++d.gemm_count;
    d.gemm_ops += 2ull * static_cast<uint64_t>(M) * static_cast<uint64_t>(W) * static_cast<uint64_t>(Kp);
    d.heavy_updates += static_cast<uint64_t>(d.gram_h) * static_cast<uint64_t>(span) *
                       static_cast<uint64_t>(std::min(bk, k_end - k0));
    g.k0 = k0;
    const bool c32 = plan->lo_bits == 32 && plan->vb == 63;  // the common split: constant shifts
    const int kc = std::min(bk, n - k0);
    const dim3 egrid((kc + 255) / 256, std::max(1, std::min(span, 148 * 32 / ((kc + 255) / 256))));
    if (plan->prec == SF_FP64)
      (c32 ? sp_gram_epilogue_kernel<double, 32, 63> : sp_gram_epilogue_kernel<double, 0, 0>)<<<egrid, 256, 0, st>>>(g);
    else
      (c32 ? sp_gram_epilogue_kernel<float, 32, 63> : sp_gram_epilogue_kernel<float, 0, 0>)<<<egrid, 256, 0, st>>>(g);
    SF_CUDA(cudaGetLastError());
    d.launches += 3;
  }
  return SF_OK;
}

sf_status sparse_prepare_lens(sf_plan* plan, DeviceState& d, const sf_problem* p) {
  const int64_t W = (plan->E + 31) / 32;
  std::vector<double> lens(static_cast<size_t>(W * 32), 0.0);
  std::copy(p->lengths, p->lengths + plan->E, lens.begin());
  SF_TRY(upload(d.lens_pad, d.dev, lens.data(), lens.size(), d.stream, "padded lengths"));
  return SF_OK;
}

sf_status sparse_prepare(sf_plan* plan, DeviceState& d, const sf_problem* p) {
  const int64_t W = (plan->E + 31) / 32;
  const int64_t n_ext = sparse_n_ext(plan->n);
  SF_TRY(d.nodebits.alloc(d.dev, static_cast<size_t>(W * n_ext) * 4, "node-packed presence bits"));
  std::vector<double> lens(static_cast<size_t>(W * 32), 0.0);
  std::copy(p->lengths, p->lengths + plan->E, lens.begin());
  SF_TRY(upload(d.lens_pad, d.dev, lens.data(), lens.size(), d.stream, "padded lengths"));
  return SF_OK;
}

template <class Real>
sf_status launch_sparse(const SparseArgs& a, cudaStream_t st) {
  using C = SparseCfg;
  using T = SparseTile<C::RK, C::RS, C::NWK, C::NWS>;
  auto* kern = stripe_sparse_kernel<Real, C::RK, C::RS, C::NWK, C::NWS>;
  SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::BYTES));
  const dim3 grid((a.n + C::TK - 1) / C::TK, (a.s_end - a.s_begin + C::TS - 1) / C::TS);
  kern<<<grid, T::NT, T::BYTES, st>>>(a);
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

template <int M, class Real, bool EXACT>
sf_status launch_wsparse_t(const WSparseArgs& a, cudaStream_t st) {
  using C = WSparseCfg;
  using T = WSparseTile<C::RK, C::RS, C::NWK, C::NWS>;
  auto* kern = stripe_wsparse_kernel<M, Real, EXACT, C::RK, C::RS, C::NWK, C::NWS>;
  SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::BYTES));
  const dim3 grid((a.n + C::TK - 1) / C::TK, (a.s_end - a.s_begin + C::TS - 1) / C::TS);
  kern<<<grid, T::NT, T::BYTES, st>>>(a);
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

template <class Real>
sf_status launch_wsparse(int metric, bool exact, const WSparseArgs& a, cudaStream_t st) {
  if (metric == SF_WEIGHTED_NORMALIZED)
    return exact ? launch_wsparse_t<kWN, Real, true>(a, st) : launch_wsparse_t<kWN, Real, false>(a, st);
  if (metric == SF_WEIGHTED_UNNORMALIZED)
    return exact ? launch_wsparse_t<kWU, Real, true>(a, st) : launch_wsparse_t<kWU, Real, false>(a, st);
  if (metric == SF_GENERALIZED)
    return exact ? launch_wsparse_t<kGen, Real, true>(a, st) : launch_wsparse_t<kGen, Real, false>(a, st);
  return fail(SF_EINVAL, "the weighted sparse walk implements the weighted metrics only");
}

// Kernel 11, per chunk: presence words + counts -> pool offsets (scan) ->
// compacted values -> wrapped columns.
sf_status wsparse_build(sf_plan* plan, DeviceState& d, int32_t C, cudaStream_t st) {
  const int n = plan->n;
  const int64_t n_ext = sparse_n_ext(n);
  const int32_t Wc = (C + 31) / 32;
  const int64_t cells = static_cast<int64_t>(Wc) * n_ext;
  ws_pack_kernel<<<grid_for(cells, 256), 256, 0, st>>>(d.emb.as<double>(), plan->row_words, C, n, Wc,
                                                        n_ext, d.wnb.as<uint32_t>(), d.wcnt.as<uint32_t>());
  size_t tmp = d.cub_bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.cubtmp.p, tmp, d.wcnt.as<uint32_t>(), d.woff.as<uint32_t>(),
                                        static_cast<int>(cells), st));
  if (plan->prec == SF_FP64)
    ws_fill_kernel<double><<<grid_for(static_cast<int64_t>(Wc) * n, 256), 256, 0, st>>>(
        d.emb.as<double>(), plan->row_words, n, Wc, n_ext, d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(),
        d.wpool.as<double>());
  else
    ws_fill_kernel<float><<<grid_for(static_cast<int64_t>(Wc) * n, 256), 256, 0, st>>>(
        d.emb.as<double>(), plan->row_words, n, Wc, n_ext, d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(),
        d.wpool.as<float>());
  ws_extend_kernel<<<grid_for(static_cast<int64_t>(Wc) * (n_ext - n), 256), 256, 0, st>>>(
      d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), n, Wc, n_ext);
  SF_CUDA(cudaGetLastError());
  d.launches += 4;
  return SF_OK;
}

template <int M, class Real, int RS = WUWalkCfg::RS>
sf_status launch_wuwalk_t(const WUWalkArgs& a, cudaStream_t st) {
  using C = WUWalkCfg;
  const dim3 grid((a.n + C::NW - 1) / C::NW, (a.s_end - a.s_begin + 32 * RS - 1) / (32 * RS));
  stripe_wuwalk_kernel<M, Real, RS, C::NW><<<grid, 32 * C::NW, 0, st>>>(a);
  SF_CUDA(cudaGetLastError());
  return SF_OK;
}

template <class Real>
sf_status launch_wuwalk(int metric, const WUWalkArgs& a, cudaStream_t st) {
  const char* v = std::getenv("SF_UWALK_VARIANT");  // A/B: 1 = 4 slots per lane, 2 = 12
  const int var = v ? std::atoi(v) : 0;
  if (metric == SF_WEIGHTED_NORMALIZED && var == 1) return launch_wuwalk_t<kWN, Real, 4>(a, st);
  if (metric == SF_WEIGHTED_NORMALIZED && var == 2) return launch_wuwalk_t<kWN, Real, 12>(a, st);
  if (metric == SF_WEIGHTED_NORMALIZED) return launch_wuwalk_t<kWN, Real>(a, st);
  if (metric == SF_WEIGHTED_UNNORMALIZED) return launch_wuwalk_t<kWU, Real>(a, st);
  if (metric == SF_GENERALIZED) return launch_wuwalk_t<kGen, Real, 4>(a, st);  // pow: fewer slots, no spills
  return fail(SF_EINVAL, "the weighted u-walk implements the weighted metrics only");
}

// Kernel 12, per chunk [r0, r0 + C): presence words + counts into the global
// arrays at word r0/32, scan, chunk total, values into the global pool at the
// running base (offsets made global), wrapped columns.
sf_status wuwalk_build(sf_plan* plan, DeviceState& d, int32_t r0, int32_t C, cudaStream_t st) {
  const int n = plan->n;
  const int64_t n_ext = sparse_n_ext(n);
  const int32_t Wc = (C + 31) / 32;
  const int64_t cells = static_cast<int64_t>(Wc) * n_ext;
  uint32_t* nb = d.wnb.as<uint32_t>() + static_cast<int64_t>(r0 / 32) * n_ext;
  uint32_t* off = d.woff.as<uint32_t>() + static_cast<int64_t>(r0 / 32) * n_ext;
  unsigned long long* base = d.wbase.as<unsigned long long>();
  ws_pack_kernel<<<grid_for(cells, 256), 256, 0, st>>>(d.emb.as<double>(), plan->row_words, C, n, Wc, n_ext,
                                                        nb, d.wcnt.as<uint32_t>());
  size_t tmp = d.cub_bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.cubtmp.p, tmp, d.wcnt.as<uint32_t>(), off, static_cast<int>(cells), st));
  wu_chunk_total_kernel<<<1, 1, 0, st>>>(off, d.wcnt.as<uint32_t>(), cells - 1, base + 1);
  const int gb = grid_for(static_cast<int64_t>(Wc) * n, 256);
  const double* lens = d.lens.as<double>() + r0;
  const bool gen = plan->metric == SF_GENERALIZED;
  if (plan->prec == SF_FP64) {
    if (gen)
      wu_fill_kernel<double, true><<<gb, 256, 0, st>>>(d.emb.as<double>(), plan->row_words, n, Wc, n_ext, nb, off,
                                                       base, lens, plan->alpha, d.wpool.as<double>(),
                                                       d.wpoola.as<double>());
    else
      wu_fill_kernel<double, false><<<gb, 256, 0, st>>>(d.emb.as<double>(), plan->row_words, n, Wc, n_ext, nb, off,
                                                        base, lens, plan->alpha, d.wpool.as<double>(), nullptr);
  } else {
    if (gen)
      wu_fill_kernel<float, true><<<gb, 256, 0, st>>>(d.emb.as<double>(), plan->row_words, n, Wc, n_ext, nb, off,
                                                      base, lens, plan->alpha, d.wpool.as<float>(),
                                                      d.wpoola.as<float>());
    else
      wu_fill_kernel<float, false><<<gb, 256, 0, st>>>(d.emb.as<double>(), plan->row_words, n, Wc, n_ext, nb, off,
                                                       base, lens, plan->alpha, d.wpool.as<float>(), nullptr);
  }
  wu_advance_base_kernel<<<1, 1, 0, st>>>(base, base + 1);
  ws_extend_kernel<<<grid_for(static_cast<int64_t>(Wc) * (n_ext - n), 256), 256, 0, st>>>(nb, off, n, Wc, n_ext);
  SF_CUDA(cudaGetLastError());
  d.launches += 6;
  return SF_OK;
}

// Heavy threshold of kernel 13 as a fraction of n (SF_WHEAVY_FRAC): a dense
// generalized term costs ~7x a weighted one (rsqrt or pow), so generalized
// keeps fewer rows dense.
double ws_heavy_frac(int metric) {
  const char* e = std::getenv("SF_WHEAVY_FRAC");
  return e ? std::atof(e) : metric == SF_GENERALIZED ? 0.6 : 0.25;
}

// Kernel 13 (wsplit_kernels.cuh), after kernel 12's build of every chunk and
// the column sums: row counts -> heavy / light split -> dense heavy rows and
// light lists -> light scatter (exact) -> dense heavy rows + epilogue.
template <class Real>
sf_status wsplit_run(sf_plan* plan, DeviceState& d, int32_t finalize, cudaStream_t st) {
  const int n = plan->n;
  const int32_t E = plan->E;
  const bool gen = plan->metric == SF_GENERALIZED;
  const bool sq = gen && plan->alpha == 0.5;  // alpha = 0.5: one rsqrt per term
  const int32_t W = (E + 31) / 32;
  const int64_t n_ext = sparse_n_ext(n);
  const uint32_t* nb = d.wnb.as<uint32_t>();
  const uint32_t* off = d.woff.as<uint32_t>();
  const Real* pool = d.wpool.as<Real>();
  const int64_t Wr = static_cast<int64_t>(W) * 32;
  // row counts and the split
  if (d.ws_cnt.bytes < static_cast<size_t>(Wr) * 4) SF_TRY(d.ws_cnt.alloc(d.dev, static_cast<size_t>(Wr) * 4, "row counts"));
  if (d.ws_hflag.bytes < static_cast<size_t>(E + 1) * 4) SF_TRY(d.ws_hflag.alloc(d.dev, static_cast<size_t>(E + 1) * 4, "heavy flags"));
  if (d.ws_hidx.bytes < static_cast<size_t>(E + 1) * 4) SF_TRY(d.ws_hidx.alloc(d.dev, static_cast<size_t>(E + 1) * 4, "heavy index"));
  if (d.ws_lcnt.bytes < static_cast<size_t>(E + 1) * 8) SF_TRY(d.ws_lcnt.alloc(d.dev, static_cast<size_t>(E + 1) * 8, "light counts"));
  if (d.ws_lptr.bytes < static_cast<size_t>(E + 1) * 8) SF_TRY(d.ws_lptr.alloc(d.dev, static_cast<size_t>(E + 1) * 8, "light rows"));
  if (d.ws_hmask.bytes < static_cast<size_t>(W) * 4) SF_TRY(d.ws_hmask.alloc(d.dev, static_cast<size_t>(W) * 4, "heavy masks"));
  if (d.ws_lmask.bytes < static_cast<size_t>(W) * 4) SF_TRY(d.ws_lmask.alloc(d.dev, static_cast<size_t>(W) * 4, "light masks"));
  if (d.ws_ccnt.bytes < static_cast<size_t>(n + 1) * 8) SF_TRY(d.ws_ccnt.alloc(d.dev, static_cast<size_t>(n + 1) * 8, "column counts"));
  if (d.ws_cptr.bytes < static_cast<size_t>(n + 1) * 8) SF_TRY(d.ws_cptr.alloc(d.dev, static_cast<size_t>(n + 1) * 8, "column lists"));
  if (d.ws_AL.bytes < static_cast<size_t>(n) * 16) SF_TRY(d.ws_AL.alloc(d.dev, static_cast<size_t>(n) * 16, "light column sums"));
  size_t t1 = 0, t2 = 0, t3 = 0;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, d.ws_hflag.as<uint32_t>(), d.ws_hidx.as<uint32_t>(), E + 1, st));
  SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, d.ws_lcnt.as<unsigned long long>(),
                                        d.ws_lptr.as<unsigned long long>(), E + 1, st));
  SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, d.ws_ccnt.as<unsigned long long>(),
                                        d.ws_cptr.as<unsigned long long>(), n + 1, st));
  const size_t tb = std::max(t1, std::max(t2, t3));
  if (d.ws_tmp.bytes < tb) SF_TRY(d.ws_tmp.alloc(d.dev, tb, "scan scratch"));
  wx_rowcount_kernel<<<std::min(W, 148 * 16), 256, 0, st>>>(nb, n_ext, n, W, E, d.ws_cnt.as<uint32_t>());
  const uint32_t thr = static_cast<uint32_t>(std::max(1.0, std::ceil(ws_heavy_frac(plan->metric) * n)));
  wx_classify_kernel<<<grid_for(Wr, 256), 256, 0, st>>>(d.ws_cnt.as<uint32_t>(), d.lens_pad.as<double>(), E, W, thr,
                                                         d.ws_hflag.as<uint32_t>(), d.ws_lcnt.as<unsigned long long>(),
                                                         d.ws_hmask.as<uint32_t>(), d.ws_lmask.as<uint32_t>());
  size_t tmp = d.ws_tmp.bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.ws_tmp.p, tmp, d.ws_hflag.as<uint32_t>(), d.ws_hidx.as<uint32_t>(), E + 1, st));
  tmp = d.ws_tmp.bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.ws_tmp.p, tmp, d.ws_lcnt.as<unsigned long long>(),
                                        d.ws_lptr.as<unsigned long long>(), E + 1, st));
  SF_CUDA(cudaGetLastError());
  uint32_t Hh = 0;
  unsigned long long LT = 0;
  SF_CUDA(cudaMemcpyAsync(&Hh, d.ws_hidx.as<uint32_t>() + E, 4, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaMemcpyAsync(&LT, d.ws_lptr.as<unsigned long long>() + E, 8, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  const int64_t H = Hh;
  const int S = n / 2;
  const int64_t ldh = (static_cast<int64_t>(n) + S + kWSK + kWSS + 64 + 3) / 4 * 4;
  const size_t w = sizeof(Real);
  const size_t uh_bytes = static_cast<size_t>(std::max<int64_t>(H, 1)) * static_cast<size_t>(ldh) * w;
  if (d.ws_UH.bytes < uh_bytes) SF_TRY(d.ws_UH.alloc(d.dev, uh_bytes, "dense heavy rows"));
  if (d.ws_LH.bytes < static_cast<size_t>(std::max<int64_t>(H, 1)) * w)
    SF_TRY(d.ws_LH.alloc(d.dev, static_cast<size_t>(std::max<int64_t>(H, 1)) * w, "heavy lengths"));
  const size_t lt = static_cast<size_t>(std::max<unsigned long long>(LT, 1));
  if (d.ws_lmid.bytes < lt * 4) SF_TRY(d.ws_lmid.alloc(d.dev, lt * 4, "light members"));
  if (d.ws_lval.bytes < lt * w) SF_TRY(d.ws_lval.alloc(d.dev, lt * w, "light member values"));
  if (gen && d.ws_lvala.bytes < lt * w) SF_TRY(d.ws_lvala.alloc(d.dev, lt * w, "light one-sided terms"));
  if (d.ws_crow.bytes < lt * 4) SF_TRY(d.ws_crow.alloc(d.dev, lt * 4, "column light rows"));
  if (d.ws_cval.bytes < lt * w) SF_TRY(d.ws_cval.alloc(d.dev, lt * w, "column light values"));
  if (d.ws_crank.bytes < lt * 4) SF_TRY(d.ws_crank.alloc(d.dev, lt * 4, "column ranks"));
  const size_t pool_entries = std::max<size_t>(d.wpool.bytes / w, 1);
  if (d.ws_prank.bytes < pool_entries * 4) SF_TRY(d.ws_prank.alloc(d.dev, pool_entries * 4, "member ranks"));
  const size_t slots = static_cast<size_t>(d.b - d.a) * static_cast<size_t>(n);
  if (d.ws_lightd.bytes < slots * 8) SF_TRY(d.ws_lightd.alloc(d.dev, slots * 8, "light part"));
  if (gen && d.ws_lightt.bytes < slots * 8) SF_TRY(d.ws_lightt.alloc(d.dev, slots * 8, "light part of the totals"));
  // dense heavy rows, light member lists, column lists
  SF_CUDA(cudaMemsetAsync(d.ws_UH.p, 0, uh_bytes, st));
  wx_heavylen_kernel<Real><<<grid_for(E, 256), 256, 0, st>>>(d.ws_hflag.as<uint32_t>(), d.ws_hidx.as<uint32_t>(),
                                                              d.lens_pad.as<double>(), E, d.ws_LH.as<Real>());
  {
    const int fb = static_cast<int>(std::min<int64_t>((W + 7) / 8, 148 * 64));
    auto fill = [&](auto* kern) {
      kern<<<fb, 256, 0, st>>>(nb, off, pool, n_ext, n, W, d.ws_hmask.as<uint32_t>(), d.ws_lmask.as<uint32_t>(),
                               d.ws_hidx.as<uint32_t>(), d.ws_lptr.as<unsigned long long>(), ldh,
                               d.lens_pad.as<double>(), plan->alpha, d.ws_UH.as<Real>(), d.ws_lmid.as<int32_t>(),
                               d.ws_lval.as<Real>(), gen ? d.ws_lvala.as<Real>() : nullptr, d.ws_prank.as<uint32_t>());
    };
    if (gen)
      fill(wx_fill_kernel<Real, true>);
    else
      fill(wx_fill_kernel<Real, false>);
  }
  if (H > 0)
    wx_extend_kernel<Real><<<grid_for(H * (ldh - n), 256), 256, 0, st>>>(d.ws_UH.as<Real>(), H, ldh, n);
  wx_colcount_kernel<<<grid_for(static_cast<int64_t>(n) * 32, 256), 256, 0, st>>>(
      nb, d.nzmask.as<uint32_t>(), d.ws_lmask.as<uint32_t>(), n_ext, n, W, d.ws_ccnt.as<unsigned long long>());
  tmp = d.ws_tmp.bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.ws_tmp.p, tmp, d.ws_ccnt.as<unsigned long long>(),
                                        d.ws_cptr.as<unsigned long long>(), n + 1, st));
  {
    auto colfill = [&](auto* kern) {
      kern<<<grid_for(static_cast<int64_t>(n) * 32, 256), 256, 0, st>>>(
          nb, off, d.nzmask.as<uint32_t>(), d.ws_lmask.as<uint32_t>(), pool, d.ws_prank.as<uint32_t>(),
          d.lens_pad.as<double>(), plan->alpha, n_ext, n, W, plan->ws_G, d.ws_cptr.as<unsigned long long>(),
          d.ws_crow.as<int32_t>(), d.ws_cval.as<Real>(), d.ws_crank.as<uint32_t>(), d.ws_AL.as<unsigned long long>());
    };
    if (gen)
      colfill(wx_colfill_kernel<Real, true>);
    else
      colfill(wx_colfill_kernel<Real, false>);
  }
  SF_CUDA(cudaGetLastError());
  // light part of every slot (exact), then the dense heavy rows + epilogue
  WSLightArgs la;
  la.cptr = d.ws_cptr.as<unsigned long long>();
  la.crow = d.ws_crow.as<int32_t>();
  la.cval = d.ws_cval.p;
  la.crank = d.ws_crank.as<uint32_t>();
  la.lptr = d.ws_lptr.as<unsigned long long>();
  la.lmid = d.ws_lmid.as<int32_t>();
  la.lval = d.ws_lval.p;
  la.lvala = gen ? d.ws_lvala.p : nullptr;
  la.alpha = plan->alpha;
  la.lightt = gen ? d.ws_lightt.as<double>() : nullptr;
  la.lens = d.lens_pad.as<double>();
  la.AL = d.ws_AL.as<unsigned long long>();
  la.n = n;
  la.s_begin = d.a;
  la.s_end = d.b;
  la.out_begin = d.a;
  const int span = d.b - d.a;
  la.G = plan->ws_G;
  la.nd = plan->ws_nd;
  const int max_tile = kWSLightSmem / (4 * la.nd * (gen ? 2 : 1));
  const int ntiles = (span + max_tile - 1) / max_tile;
  la.tile = (span + ntiles - 1) / ntiles;
  la.lightd = d.ws_lightd.as<double>();
  la.pairs = d.exec_ctr.as<unsigned long long>();
  const size_t lsmem = static_cast<size_t>(la.nd) * static_cast<size_t>(la.tile) * 4 * (gen ? 2 : 1);
  auto light = [&](auto* kern) -> sf_status {
    SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lsmem)));
    kern<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(ntiles)), kWSLightThreads, lsmem, st>>>(la);
    return SF_OK;
  };
  // digit planes: 16 bits each, from the lengths' range (plan time);
  // -1 weighted, 0 generalized (pow), 1 generalized alpha = 0.5 (rsqrt)
  auto by_nd = [&](auto genc) -> sf_status {
    constexpr int GA = decltype(genc)::value;
    switch (la.nd) {
      case 4: return light(wx_light_kernel<Real, 4, GA>);
      case 5: return light(wx_light_kernel<Real, 5, GA>);
      case 6: return light(wx_light_kernel<Real, 6, GA>);
      case 7: return light(wx_light_kernel<Real, 7, GA>);
      default: return light(wx_light_kernel<Real, 8, GA>);
    }
  };
  if (!gen)
    SF_TRY(by_nd(std::integral_constant<int, -1>{}));
  else if (sq)
    SF_TRY(by_nd(std::integral_constant<int, 1>{}));
  else
    SF_TRY(by_nd(std::integral_constant<int, 0>{}));
  SF_CUDA(cudaGetLastError());
  WSDenseArgs da;
  da.UH = d.ws_UH.p;
  da.LH = d.ws_LH.p;
  da.H = H;
  da.ldh = ldh;
  da.n = n;
  da.s_begin = d.a;
  da.s_end = d.b;
  da.out_begin = d.a;
  da.finalize = finalize ? 1 : 0;
  da.lightd = d.ws_lightd.as<double>();
  da.lightt = gen ? d.ws_lightt.as<double>() : nullptr;
  da.alpha = plan->alpha;
  da.A = d.wA.as<double2>();
  da.dist = d.dist.p;
  da.tot = plan->metric == SF_WEIGHTED_UNNORMALIZED ? nullptr : d.tot.p;
  while (d.gemm_ev.size() < 2 * (d.gemm_count + 1)) {
    cudaEvent_t e;
    SF_CUDA(cudaEventCreate(&e));
    d.gemm_ev.push_back(e);
  }
  auto dense = [&](auto* kern, int kt) -> sf_status {
    const size_t dsmem = (2 * kWSR * (2 * static_cast<size_t>(kt) + kWSS) + 2 * kWSR) * w;
    const dim3 dgrid(static_cast<unsigned>((n + kt - 1) / kt), static_cast<unsigned>((span + kWSS - 1) / kWSS));
    SF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsmem)));
    SF_CUDA(cudaEventRecord(d.gemm_ev[2 * d.gemm_count], st));
    kern<<<dgrid, kWSThreads, dsmem, st>>>(da);
    return SF_OK;
  };
  if (plan->metric == SF_WEIGHTED_UNNORMALIZED)
    SF_TRY(dense(wx_dense_kernel<kWU, Real, false>, wx_dense_kt<kWU>()));
  else if (!gen)
    SF_TRY(dense(wx_dense_kernel<kWN, Real, false>, wx_dense_kt<kWN>()));
  else if (sq)
    SF_TRY(dense(wx_dense_kernel<kGen, Real, true>, wx_dense_kt<kGen>()));
  else
    SF_TRY(dense(wx_dense_kernel<kGen, Real, false>, wx_dense_kt<kGen>()));
  SF_CUDA(cudaGetLastError());
  SF_CUDA(cudaEventRecord(d.gemm_ev[2 * d.gemm_count + 1], st));
  ++d.gemm_count;
  const uint64_t live = static_cast<uint64_t>(span) * static_cast<uint64_t>(n);
  // FP64-pipe instructions per (heavy row, slot), from the kernels' SASS:
  // DADD + DFMA (WN/WU); 14 for generalized alpha = 0.5 (DADD x3, DSETP x2,
  // DMUL x4, DFMA x5 around one MUFU.RSQ64H); the pow path is not counted
  const uint64_t per = gen ? (sq ? 14ull : 0ull) : 2ull;
  d.host_fp64_ops += per * static_cast<uint64_t>(H) * live;
  d.heavy_updates += static_cast<uint64_t>(H) * live;
  d.launches += 14;
  return SF_OK;
}

// Upper bound of the present (row, sample) entries: a row has at most
// min(n, table entries under it) nonzero samples.
uint64_t present_bound(const sf_problem* p) {
  const int E = p->n_rows;
  std::vector<uint64_t> c(static_cast<size_t>(E), 0);
  uint64_t total = 0;
  for (int r = 0; r < E; ++r) {  // postorder: children before parents
    const int f = p->leaf_feature[r];
    if (f >= 0) c[static_cast<size_t>(r)] += static_cast<uint64_t>(p->feat_ptr[f + 1] - p->feat_ptr[f]);
    total += std::min<uint64_t>(c[static_cast<size_t>(r)], static_cast<uint64_t>(p->n_samples));
    const int par = p->parent_row[r];
    if (par >= 0) c[static_cast<size_t>(par)] += c[static_cast<size_t>(r)];
  }
  return total;
}

// Layout of one chunk's schedule arrays inside the packed device buffer.
enum { kLeafRows, kLeafFeat, kIntRows, kCptr, kCodes, kCarrySrc, kCarryDst, kNumArr };

// Kernel 13's sparse value build (wsplit_kernels.cuh): from the chunk's
// presence bit rows (K1, every row in one chunk) to the presence words, pool
// offsets and the value pool of the chunked build — without dense value rows.
template <class Real, class Arr>
sf_status wx_values_build(sf_plan* plan, DeviceState& d, const Chunk& c, Arr arr, cudaStream_t st) {
  const int n = plan->n;
  const int32_t E = plan->E;
  const int32_t W = (E + 31) / 32;
  const int64_t n_ext = sparse_n_ext(n);
  const int64_t RW = plan->row_words;
  const int64_t cells = static_cast<int64_t>(W) * n_ext;
  uint32_t* nb = d.wnb.as<uint32_t>();
  uint32_t* off = d.woff.as<uint32_t>();
  wx_words_kernel<<<grid_for(cells, 256), 256, 0, st>>>(d.emb.as<uint32_t>(), RW, E, n, W, n_ext, nb,
                                                         d.wcnt.as<uint32_t>());
  size_t tmp = d.cub_bytes;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(d.cubtmp.p, tmp, d.wcnt.as<uint32_t>(), off, static_cast<int>(cells), st));
  // the pool's size (fp32: the cast below)
  wu_chunk_total_kernel<<<1, 1, 0, st>>>(off, d.wcnt.as<uint32_t>(), cells - 1, d.wbase.as<unsigned long long>());
  ws_extend_kernel<<<grid_for(static_cast<int64_t>(W) * (n_ext - n), 256), 256, 0, st>>>(nb, off, n, W, n_ext);
  double* pool64 = nullptr;
  if (sizeof(Real) == 8) {
    pool64 = d.wpool.as<double>();
  } else {
    const size_t need = d.wpool.bytes / sizeof(Real) * 8;
    if (d.ws_pool64.bytes < need) SF_TRY(d.ws_pool64.alloc(d.dev, need, "fp64 value pool"));
    pool64 = d.ws_pool64.as<double>();
  }
  const int nl = static_cast<int>(c.leaf_rows.size());
  if (nl > 0)
    wx_leaf_values_kernel<<<grid_for(static_cast<int64_t>(nl) * 32, 256), 256, 0, st>>>(
        pool64, nb, off, n_ext, arr(kLeafRows), arr(kLeafFeat), nl, d.feat_ptr.as<int64_t>(), d.sidx.as<int32_t>(),
        d.counts.as<double>(), d.totals.as<double>());
  for (size_t h = 0; h + 1 < c.lvl_ptr.size(); ++h) {
    const int lo = c.lvl_ptr[h], hi = c.lvl_ptr[h + 1];
    if (hi <= lo) continue;
    wx_level_values_kernel<<<grid_for(static_cast<int64_t>(hi - lo) * RW, 256), 256, 0, st>>>(
        pool64, d.emb.as<uint32_t>(), RW, nb, off, n_ext, arr(kIntRows) + lo, arr(kCptr) + lo, arr(kCodes), hi - lo);
    d.launches++;
  }
  if (sizeof(Real) == 4)
    wx_pool_to_float_kernel<<<grid_for(static_cast<int64_t>(d.wpool.bytes / sizeof(Real)), 256), 256, 0, st>>>(
        pool64, d.wbase.as<unsigned long long>(), d.wpool.as<float>());
  if (plan->metric == SF_GENERALIZED && d.wpoola.p)  // the u-walk fallback's second pool
    wx_poola_kernel<Real><<<grid_for(static_cast<int64_t>(W) * n, 256), 256, 0, st>>>(
        nb, off, n_ext, n, W, d.lens_pad.as<double>(), plan->alpha, d.wpool.as<Real>(), d.wpoola.as<Real>());
  SF_CUDA(cudaGetLastError());
  d.launches += 6;
  return SF_OK;
}


sf_status upload_schedule(DeviceState& d, const Schedule& s) {
  std::vector<int32_t> packed;
  d.sched_off.clear();
  for (const Chunk& c : s.chunks) {
    const std::vector<int32_t>* arrs[kNumArr] = {&c.leaf_rows, &c.leaf_feat, &c.int_rows, &c.cptr,
                                                 &c.codes, &c.carry_src, &c.carry_dst};
    for (auto* v : arrs) {
      d.sched_off.push_back(static_cast<int64_t>(packed.size()));
      packed.insert(packed.end(), v->begin(), v->end());
      while (packed.size() % 4) packed.push_back(0);  // 16-byte alignment
    }
  }
  return upload(d.sched, d.dev, packed.data(), packed.size(), d.stream, "schedule");
}

// host_d / host_t (optional): this device's slice of the caller's output.
// With the split kernel the stripes are then computed in chunks and each
// chunk's D2H copy runs on a second stream while the next chunk computes.
sf_status run_device(sf_plan* plan, DeviceState& d, int32_t finalize, void* host_d = nullptr,
                     void* host_t = nullptr) {
  SF_CUDA(cudaSetDevice(d.dev));
  const bool dbg = std::getenv("SF_DEBUG") != nullptr;
  const auto t_run = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (dbg)
      std::fprintf(stderr, "stripefrac:   run dev %d %s at %.1f ms (host)\n", d.dev, what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_run).count());
  };
  const cudaStream_t st = d.stream;
  const int n = plan->n;
  const int64_t rows_here = d.b - d.a;
  const size_t w = plan->prec == SF_FP64 ? 8 : 4;
  const int64_t slots = rows_here * n;
  // events: [0]=start, per chunk (embed start, stripe start, stripe end), fin start, fin end
  const size_t need_ev = 3 + 3 * plan->sched.chunks.size();
  while (d.events.size() < need_ev) {
    cudaEvent_t e;
    SF_CUDA(cudaEventCreate(&e));
    d.events.push_back(e);
  }
  SF_CUDA(cudaEventRecord(d.events[0], st));
  d.gemm_count = 0;
  d.gemm_ops = 0;
  d.heavy_updates = 0;
  d.host_fp64_ops = 0;
  if (plan->kernel != 10 && plan->kernel != 12 && plan->kernel != 13) {  // these kernels write every slot
    SF_CUDA(cudaMemsetAsync(d.dist.p, 0, static_cast<size_t>(slots) * w, st));
    if (d.tot.p && plan->metric != SF_WEIGHTED_UNNORMALIZED)
      SF_CUDA(cudaMemsetAsync(d.tot.p, 0, static_cast<size_t>(slots) * w, st));
  }
  SF_CUDA(cudaMemsetAsync(d.exec_ctr.p, 0, 2 * sizeof(unsigned long long), st));

  const int64_t stride = plan->row_words;
  const int ncols = static_cast<int>((plan->bits || plan->wbits) ? (n + 31) / 32 : n);
  const int32_t* base = d.sched.as<int32_t>();
  for (size_t ci = 0; ci < plan->sched.chunks.size(); ++ci) {
    const Chunk& c = plan->sched.chunks[ci];
    auto arr = [&](int k) { return base + d.sched_off[ci * kNumArr + static_cast<size_t>(k)]; };
    const int C = c.r1 - c.r0;
    SF_CUDA(cudaEventRecord(d.events[1 + 3 * ci], st));
    // ---- K1: embedding rows of this chunk (bit rows: unweighted presence, or
    // the weighted rows' presence for the sparse value build)
    const bool bitrows = plan->bits || plan->wbits;
    const size_t row_bytes = static_cast<size_t>(stride) * (bitrows ? 4 : 8);
    SF_CUDA(cudaMemsetAsync(d.emb.p, 0, row_bytes * static_cast<size_t>(C), st));
    const int nl = static_cast<int>(c.leaf_rows.size());
    if (nl > 0) {
      const int blocks = grid_for(static_cast<int64_t>(nl) * 32, 256);
      if (plan->bits)
        embed_leaf_bits<<<blocks, 256, 0, st>>>(d.emb.as<uint32_t>(), stride, arr(kLeafRows),
                                                arr(kLeafFeat), nl, d.feat_ptr.as<int64_t>(),
                                                d.sidx.as<int32_t>(), d.counts.as<double>());
      else if (plan->wbits)
        wx_leaf_bits_kernel<<<blocks, 256, 0, st>>>(d.emb.as<uint32_t>(), stride, arr(kLeafRows), arr(kLeafFeat),
                                                    nl, d.feat_ptr.as<int64_t>(), d.sidx.as<int32_t>(),
                                                    d.counts.as<double>(), d.totals.as<double>());
      else
        embed_leaf_values<<<blocks, 256, 0, st>>>(d.emb.as<double>(), stride, arr(kLeafRows),
                                                  arr(kLeafFeat), nl, d.feat_ptr.as<int64_t>(),
                                                  d.sidx.as<int32_t>(), d.counts.as<double>(),
                                                  d.totals.as<double>());
      SF_CUDA(cudaGetLastError());
      d.launches++;
    }
    for (size_t h = 0; h + 1 < c.lvl_ptr.size(); ++h) {
      const int lo = c.lvl_ptr[h], hi = c.lvl_ptr[h + 1];
      if (hi <= lo) continue;
      const dim3 grid((ncols + 127) / 128, std::min(hi - lo, 65535));
      if (bitrows)
        embed_level_bits<<<grid, 128, 0, st>>>(d.emb.as<uint32_t>(), stride, d.pend.as<uint32_t>(),
                                               arr(kIntRows) + lo, arr(kCptr) + lo, arr(kCodes),
                                               hi - lo, ncols);
      else
        embed_level_values<<<grid, 128, 0, st>>>(d.emb.as<double>(), stride, d.pend.as<double>(),
                                                 arr(kIntRows) + lo, arr(kCptr) + lo, arr(kCodes),
                                                 hi - lo, ncols);
      SF_CUDA(cudaGetLastError());
      d.launches++;
    }
    if (plan->wbits) {
      SF_TRY(plan->prec == SF_FP64 ? wx_values_build<double>(plan, d, c, arr, st)
                                   : wx_values_build<float>(plan, d, c, arr, st));
    } else if (plan->kernel == 12 || plan->kernel == 13) {
      if (ci == 0) SF_CUDA(cudaMemsetAsync(d.wbase.p, 0, 16, st));
      SF_TRY(wuwalk_build(plan, d, c.r0, C, st));
    } else if (plan->kernel == 11) {
      SF_TRY(wsparse_build(plan, d, C, st));
    } else if (plan->kernel == 10) {
      phase("embedding enqueued");
      // with the tensor-core heavy path the column-owned light kernel runs per
      // column group, right before that group's GEMM blocks, so each group's
      // stripes are final (and copied out) while later groups compute
      d.defer_light = d.banded && d.light_columns && heavy_gemm_enabled();
      SF_TRY(split_build(plan, d, st));
      phase("split prep + first light pass enqueued");
    } else if (plan->kernel == 2) {
      // node-packed presence bits for the sparse walk
      const int64_t W = (plan->E + 31) / 32;
      const int64_t n_ext = sparse_n_ext(n);
      transpose_bits_kernel<<<grid_for(W * stride * 32, 256), 256, 0, st>>>(
          d.emb.as<uint32_t>(), stride, plan->E, n, d.nodebits.as<uint32_t>(), n_ext,
          static_cast<int32_t>(W));
      extend_columns_kernel<<<grid_for(W * (n_ext - n), 256), 256, 0, st>>>(
          d.nodebits.as<uint32_t>(), n_ext, n, static_cast<int32_t>(W));
      SF_CUDA(cudaGetLastError());
      d.launches += 2;
    }
    SF_CUDA(cudaEventRecord(d.events[2 + 3 * ci], st));
    // ---- K2: stripe update over the chunk's rows
    if (plan->kernel == 12 || plan->kernel == 13) {
      if (ci + 1 == plan->sched.chunks.size()) {  // every row is resident now: one pass
        const int64_t n_ext = sparse_n_ext(n);
        const int32_t W = (plan->E + 31) / 32;
        const bool gen = plan->metric == SF_GENERALIZED;
        const int gb = (n + 31) / 32;  // wu_colsum_kernel: 32 columns per block
        if (plan->prec == SF_FP64) {
          if (gen)
            wu_colsum_kernel<double, true><<<gb, 32 * kColParts, 0, st>>>(d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), n_ext, n, W,
                                                               d.lens_pad.as<double>(), d.wpool.as<double>(),
                                                               d.wpoola.as<double>(), d.wA.as<double2>());
          else
            wu_colsum_kernel<double, false><<<gb, 32 * kColParts, 0, st>>>(d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), n_ext, n, W,
                                                                d.lens_pad.as<double>(), d.wpool.as<double>(),
                                                                nullptr, d.wA.as<double2>());
        } else {
          if (gen)
            wu_colsum_kernel<float, true><<<gb, 32 * kColParts, 0, st>>>(d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), n_ext, n, W,
                                                              d.lens_pad.as<double>(), d.wpool.as<float>(),
                                                              d.wpoola.as<float>(), d.wA.as<double2>());
          else
            wu_colsum_kernel<float, false><<<gb, 32 * kColParts, 0, st>>>(d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), n_ext, n, W,
                                                               d.lens_pad.as<double>(), d.wpool.as<float>(),
                                                               nullptr, d.wA.as<double2>());
        }
        wu_nzmask_kernel<<<grid_for(static_cast<int64_t>((W + 31) / 32) * n, 256), 256, 0, st>>>(
            d.wnb.as<uint32_t>(), n_ext, n, W, d.nzmask.as<uint32_t>());
        bool uwalk = plan->kernel == 12;
        if (plan->kernel == 13) {
          // without the memory for its dense rows / light lists the weighted
          // split hands the run to the u-walk (same tolerance, no extra memory)
          const sf_status ws = plan->prec == SF_FP64 ? wsplit_run<double>(plan, d, finalize, st)
                                                     : wsplit_run<float>(plan, d, finalize, st);
          if (ws == SF_ENOMEM) {
            cudaGetLastError();
            if (std::getenv("SF_DEBUG"))
              std::fprintf(stderr, "stripefrac: device %d: %s; weighted rows on the u-walk\n", d.dev, sf::last_error());
            uwalk = true;
          } else {
            SF_TRY(ws);
          }
        }
        if (uwalk) {
          // combined cells (SF_UWALK_NBO=0: separate word / offset arrays)
          const char* nbo_env = std::getenv("SF_UWALK_NBO");
          const int64_t cells = static_cast<int64_t>(W) * n_ext;
          bool use_nbo = !(nbo_env && std::atoi(nbo_env) == 0);
          if (use_nbo && d.wnbo.bytes < static_cast<size_t>(cells) * 8)
            use_nbo = d.wnbo.alloc(d.dev, static_cast<size_t>(cells) * 8, "word/offset cells") == SF_OK;
          cudaGetLastError();
          if (use_nbo)
            wu_combine_kernel<<<grid_for(cells, 256), 256, 0, st>>>(d.wnb.as<uint32_t>(), d.woff.as<uint32_t>(), cells,
                                                                     d.wnbo.as<unsigned long long>());
          SF_CUDA(cudaGetLastError());
          WUWalkArgs a;
          a.nbo = use_nbo ? d.wnbo.as<unsigned long long>() : nullptr;
          const char* lst = std::getenv("SF_UWALK_LIST");
          a.nz = (lst && std::atoi(lst) == 0) ? nullptr : d.nzmask.as<uint32_t>();
          a.nb = d.wnb.as<uint32_t>();
          a.off = d.woff.as<uint32_t>();
          a.pool = d.wpool.p;
          a.poola = d.wpoola.p;
          a.lens = d.lens_pad.as<double>();
          a.A = d.wA.as<double2>();
          a.n_ext = n_ext;
          a.W = W;
          a.n = n;
          a.s_begin = d.a;
          a.s_end = d.b;
          a.out_begin = d.a;
          a.finalize = finalize ? 1 : 0;
          a.alpha = plan->alpha;
          a.dist = d.dist.p;
          a.tot = plan->metric == SF_WEIGHTED_UNNORMALIZED ? nullptr : d.tot.p;
          a.exec_updates = d.exec_ctr.as<unsigned long long>();
          a.fp64_ops = d.exec_ctr.as<unsigned long long>() + 1;
          SF_TRY(plan->prec == SF_FP64 ? launch_wuwalk<double>(plan->metric, a, st)
                                       : launch_wuwalk<float>(plan->metric, a, st));
          d.launches++;
        }
        const int S = n / 2;
        if (n % 2 == 0 && S - 1 >= d.a && S - 1 < d.b) {  // duplicated half stripe
          const int64_t row_off = static_cast<int64_t>(S - 1 - d.a) * n;
          const bool has_tot = plan->metric != SF_WEIGHTED_UNNORMALIZED;
          if (plan->prec == SF_FP64)
            wu_mirror_kernel<double><<<grid_for(S, 256), 256, 0, st>>>(d.dist.as<double>(), has_tot ? d.tot.as<double>() : nullptr, n, row_off);
          else
            wu_mirror_kernel<float><<<grid_for(S, 256), 256, 0, st>>>(d.dist.as<float>(), has_tot ? d.tot.as<float>() : nullptr, n, row_off);
          SF_CUDA(cudaGetLastError());
          d.launches++;
        }
      } else {
        d.launches--;  // nothing launched for this chunk
      }
    } else if (plan->kernel == 11) {
      WSparseArgs a;
      a.nb = d.wnb.as<uint32_t>();
      a.off = d.woff.as<uint32_t>();
      a.pool = d.wpool.p;
      a.n_ext = sparse_n_ext(n);
      a.lens = d.lens.as<double>() + c.r0;
      a.C = C;
      a.Wc = (C + 31) / 32;
      a.n = n;
      a.s_begin = d.a;
      a.s_end = d.b;
      a.dist = d.dist.p;
      a.tot = plan->metric == SF_WEIGHTED_UNNORMALIZED ? nullptr : d.tot.p;
      a.exec_updates = d.exec_ctr.as<unsigned long long>();
      a.alpha = plan->alpha;
      SF_TRY(plan->prec == SF_FP64 ? launch_wsparse<double>(plan->metric, plan->exact, a, st)
                                   : launch_wsparse<float>(plan->metric, plan->exact, a, st));
    } else if (plan->kernel == 10) {
      SplitArgs a;
      a.nx = d.nodebits.as<unsigned long long>();
      a.limbs = d.limbs.as<double2>();
      a.n_heavy = d.nheavy.as<unsigned int>();
      a.gl = d.lightsum.as<unsigned long long>();
      a.colsum = d.colsum.as<unsigned long long>();
      a.cacc = d.cacc.as<unsigned long long>();
      a.n_ext = sparse_n_ext(n);
      a.n = n;
      a.out_begin = d.a;
      a.lo_bits = plan->lo_bits;
      a.scale = plan->scale;
      a.finalize = finalize ? 1 : 0;
      a.dist = d.dist.p;
      a.tot = d.tot.p;
      a.counters = d.exec_ctr.as<unsigned long long>();
      a.levels = plan->levels;
      a.vb = plan->vb;
      a.dacc = plan->levels > 1 ? d.deepsum.as<unsigned long long>() : nullptr;
      a.dcolsum = plan->levels > 1 ? d.dcolsum.as<unsigned long long>() : nullptr;
      a.dcacc = plan->levels > 1 ? d.dcacc.as<unsigned long long>() : nullptr;
      // light-sum passes (one unless memory is short); within a pass, with a
      // host destination, chunks of whole 512-stripe tiles whose D2H copy
      // overlaps the next chunk's compute
      const int tile = 32 * SplitCfg::RS;
      bool gram = heavy_gemm_enabled();
      if (gram) {
        // the tensor-core operands are sized by the heavy-row count, known
        // only now; without the memory for them the DFMA heavy walk (the
        // same exact sums, bit for bit) takes the heavy rows
        const sf_status gs = gram_prepare(plan, d, st);
        phase("tensor-core operands prepared");
        if (gs == SF_ENOMEM) {
          gram = false;
          cudaGetLastError();
          if (std::getenv("SF_DEBUG"))
            std::fprintf(stderr, "stripefrac: device %d: %s; heavy rows on the DFMA walk\n", d.dev, sf::last_error());
        } else {
          SF_TRY(gs);
        }
      }
      if (d.light_lazy) {
        if (!d.light_sized) {
          // the light sums next to the GEMM operands still to come (gram_run)
          size_t extra = 0;
          if (gram) {
            const int span_all = d.b - d.a;
            const int64_t bk = gram_block(span_all);
            const int64_t M = bk * d.gram_nd;
            extra = static_cast<size_t>(M * d.gram_kp) + static_cast<size_t>(M * (span_all + bk - 1)) * 4;
          }
          SF_TRY(light_sums_alloc(plan, d, extra));
          d.light_sized = true;
        }
        // the first pass's deeper-level sums (split_build left them for now)
        const int p1 = std::min(d.b, d.a + d.light_pass);
        if (plan->levels > 1) {
          SF_CUDA(cudaMemsetAsync(d.deepsum.p, 0,
                                  static_cast<size_t>(p1 - d.a) * n * 16 * static_cast<size_t>(plan->levels - 1), st));
          SF_TRY(split_scatter_deep(plan, d, st, d.a, p1, true));
        }
        a.gl = d.lightsum.as<unsigned long long>();
        a.dacc = plan->levels > 1 ? d.deepsum.as<unsigned long long>() : nullptr;
      }
      if (!gram && d.defer_light) {  // the DFMA walk expects the whole pass's light sums first
        d.defer_light = false;
        SF_TRY(light_columns_run(plan, d, st, d.a, std::min(d.b, d.a + d.light_pass), 0, n));
      }
      int ci = 0;
      if (host_d && !d.copy_stream) SF_CUDA(cudaStreamCreateWithFlags(&d.copy_stream, cudaStreamNonBlocking));
      // a finished block: event, then its D2H copy on the copy stream (or,
      // pageable destinations, recorded for the caller's staged copies)
      auto finished = [&](int r0, int r1, int k0, int k1) -> sf_status {
        if (!host_d) return SF_OK;
        while (static_cast<int>(d.chunk_events.size()) <= ci) {
          cudaEvent_t e;
          SF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          d.chunk_events.push_back(e);
        }
        SF_CUDA(cudaEventRecord(d.chunk_events[static_cast<size_t>(ci)], st));
        const DeviceState::Span sp{r0 - d.a, r1 - r0, k0, k1 - k0};
        ++ci;
        if (d.defer_copy) {
          d.chunk_spans.push_back(sp);
          return SF_OK;
        }
        SF_CUDA(cudaStreamWaitEvent(d.copy_stream, d.chunk_events[static_cast<size_t>(ci - 1)], 0));
        const size_t pitch = static_cast<size_t>(n) * w;
        const size_t off = static_cast<size_t>(sp.row0) * pitch + static_cast<size_t>(sp.col0) * w;
        SF_CUDA(cudaMemcpy2DAsync(static_cast<char*>(host_d) + off, pitch, d.dist.as<char>() + off, pitch,
                                  static_cast<size_t>(sp.cols) * w, static_cast<size_t>(sp.rows),
                                  cudaMemcpyDeviceToHost, d.copy_stream));
        if (host_t)
          SF_CUDA(cudaMemcpy2DAsync(static_cast<char*>(host_t) + off, pitch, d.tot.as<char>() + off, pitch,
                                    static_cast<size_t>(sp.cols) * w, static_cast<size_t>(sp.rows),
                                    cudaMemcpyDeviceToHost, d.copy_stream));
        return SF_OK;
      };
      auto deep_epilogue = [&](int c0, int c1, int k0, int k1) -> sf_status {
        if (plan->levels <= 1) return SF_OK;  // lengths off the main grid: exact multi-level epilogue
        a.s_begin = c0;
        a.s_end = c1;
        a.k_begin = k0;
        a.k_end = k1;
        const int blocks = grid_for(static_cast<int64_t>(c1 - c0) * (k1 - k0), 256);
        if (plan->prec == SF_FP64)
          sp_deep_epilogue_kernel<double><<<blocks, 256, 0, st>>>(a);
        else
          sp_deep_epilogue_kernel<float><<<blocks, 256, 0, st>>>(a);
        SF_CUDA(cudaGetLastError());
        d.launches++;
        return SF_OK;
      };
      for (int p0 = d.a; p0 < d.b; p0 += d.light_pass) {
        const int p1 = std::min(d.b, p0 + d.light_pass);
        if (p0 != d.a) SF_TRY(split_scatter(plan, d, st, p0, p1, false));
        a.gl_begin = p0;
        const int span = p1 - p0;
        if (gram) {
          // the GEMM blocks run along the u columns over the whole pass; with
          // a host destination, every group of blocks (a column strip of the
          // pass's stripes) is copied while the next group computes
          const int bk = gram_block(span);
          const char* cg = std::getenv("SF_COPY_GROUPS");  // A/B: column strips per pass
          const int gmax = cg ? std::max(1, std::atoi(cg)) : 12;
          const int ngrp = host_d ? std::max(1, std::min(gmax, n / (2 * bk))) : 1;
          const int gw = ((n + ngrp - 1) / ngrp + bk - 1) / bk * bk;
          // the first strip is one GEMM block wide, so its copy starts early
          // (the D2H of 5 GB at C3 is as long as the compute it overlaps)
          for (int k0 = 0, k1 = 0; k0 < n; k0 = k1) {
            k1 = std::min(n, k0 + (k0 == 0 && ngrp > 1 ? bk : gw));
            if (d.defer_light) SF_TRY(light_columns_run(plan, d, st, p0, p1, k0, k1));
            SF_TRY(gram_run(plan, d, p0, p1, p0, finalize, st, k0, k1));
            if (plan->levels > 2) SF_TRY(deep_epilogue(p0, p1, k0, k1));  // two levels: fused in the epilogue
            SF_TRY(finished(p0, p1, k0, k1));
          }
          continue;
        }
        // DFMA heavy walk: chunks of whole 512-stripe tiles
        const int nch = host_d ? std::max(1, std::min(8, span / (4 * tile))) : 1;
        const int per = (span + nch - 1) / nch;
        const int step = (per + tile - 1) / tile * tile;
        for (int c0 = p0; c0 < p1; c0 += step) {
          const int c1 = std::min(p1, c0 + step);
          a.s_begin = c0;
          a.s_end = c1;
          SF_TRY(plan->prec == SF_FP64 ? launch_split<double>(a, st) : launch_split<float>(a, st));
          d.launches++;
          SF_TRY(deep_epilogue(c0, c1, 0, n));
          SF_TRY(finished(c0, c1, 0, n));
        }
      }
      d.launches--;  // counted once more below
      phase("heavy rows + copies enqueued");
    } else if (plan->kernel == 2) {
      SparseArgs a;
      a.nb = d.nodebits.as<uint32_t>();
      a.n_ext = sparse_n_ext(n);
      a.lens = d.lens_pad.as<double>();
      a.W = static_cast<int32_t>((plan->E + 31) / 32);
      a.n = n;
      a.s_begin = d.a;
      a.s_end = d.b;
      a.dist = d.dist.p;
      a.tot = d.tot.p;
      a.exec_updates = d.exec_ctr.as<unsigned long long>();
      SF_TRY(plan->prec == SF_FP64 ? launch_sparse<double>(a, st) : launch_sparse<float>(a, st));
    } else {
      StripeArgs a;
      a.emb = d.emb.p;
      a.row_stride = stride;
      a.lens = d.lens.as<double>() + c.r0;
      a.C = C;
      a.n = n;
      a.s_begin = d.a;
      a.s_end = d.b;
      a.dist = d.dist.p;
      a.tot = plan->metric == SF_WEIGHTED_UNNORMALIZED ? nullptr : d.tot.p;
      a.exec_updates = d.exec_ctr.as<unsigned long long>();
      SF_TRY(launch_stripes(plan->metric, plan->prec, plan->bits ? kSrcBits : kSrcF64,
                            plan->exact, a, st));
    }
    d.launches++;
    SF_CUDA(cudaEventRecord(d.events[3 + 3 * ci], st));
    const int ncarry = static_cast<int>(c.carry_src.size());
    if (ncarry > 0) {
      const dim3 grid((ncols + 127) / 128, std::min(ncarry, 65535));
      if (plan->bits)
        embed_carry<uint32_t><<<grid, 128, 0, st>>>(d.emb.as<uint32_t>(), d.pend.as<uint32_t>(),
                                                    stride, arr(kCarrySrc), arr(kCarryDst),
                                                    ncarry, ncols);
      else
        embed_carry<double><<<grid, 128, 0, st>>>(d.emb.as<double>(), d.pend.as<double>(), stride,
                                                  arr(kCarrySrc), arr(kCarryDst), ncarry, ncols);
      SF_CUDA(cudaGetLastError());
      d.launches++;
    }
  }
  const size_t ne = d.events.size();
  SF_CUDA(cudaEventRecord(d.events[ne - 2], st));
  if (finalize && plan->metric != SF_WEIGHTED_UNNORMALIZED && (plan->kernel <= 2 || plan->kernel == 11)) {
    const int blocks = grid_for(slots, 256);
    if (plan->prec == SF_FP64)
      finalize_kernel<double><<<blocks, 256, 0, st>>>(d.dist.as<double>(), d.tot.as<double>(), slots);
    else
      finalize_kernel<float><<<blocks, 256, 0, st>>>(d.dist.as<float>(), d.tot.as<float>(), slots);
    SF_CUDA(cudaGetLastError());
    d.launches++;
  }
  SF_CUDA(cudaEventRecord(d.events[ne - 1], st));
  return SF_OK;
}

// fn(DeviceState&) for every device of the plan, one host thread per device
// when there are several (their enqueues, synchronous steps and host copies
// then overlap); the first failure's status and message are returned on the
// calling thread (sf_last_error is thread-local).
template <class F>
sf_status for_each_device(sf_plan* plan, F&& fn) {
  const size_t G = plan->devs.size();
  if (G == 1) return fn(*plan->devs[0]);
  std::vector<sf_status> st(G, SF_OK);
  std::vector<std::string> err(G);
  std::vector<std::thread> th;
  for (size_t i = 0; i < G; ++i)
    th.emplace_back([&, i] {
      st[i] = fn(*plan->devs[i]);
      if (st[i] != SF_OK) err[i] = sf::last_error();
    });
  for (auto& t : th) t.join();
  for (size_t i = 0; i < G; ++i)
    if (st[i] != SF_OK) return fail(st[i], err[i]);
  return SF_OK;
}

// ------------------------------------------------------------ pageable downloads
// A D2H cudaMemcpy into pageable memory goes through the driver's small
// staging buffers on one thread (C3: ~16 GB/s, 0.3 s of a 0.77 s call).
// Pageable destinations instead get a process-wide pinned double buffer:
// block b+1 is copied device -> pinned while host threads copy block b
// pinned -> destination (the reference hands out pageable Eigen buffers).
bool host_pinned(const void* ptr) {
  cudaPointerAttributes at{};
  if (!ptr || cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

struct PinnedStaging {
  std::mutex mu;
  char* slot[2] = {nullptr, nullptr};
  size_t bytes = 0;
};
// one double buffer per device, so several devices download in parallel
PinnedStaging& staging(int device) {
  static PinnedStaging s[64];  // freed at process exit by the driver
  return s[device & 63];
}

void parallel_memcpy(char* dst, const char* src, size_t bytes, unsigned max_threads) {
  const size_t min_piece = 8ull << 20;
  size_t T = std::min<size_t>(std::max(1u, max_threads), std::max<size_t>(1, bytes / min_piece));
  if (T <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t piece = (bytes + T - 1) / T;
  std::vector<std::thread> th;
  for (size_t i = 1; i < T; ++i) {
    const size_t o = i * piece;
    if (o >= bytes) break;
    th.emplace_back([=] { std::memcpy(dst + o, src + o, std::min(piece, bytes - o)); });
  }
  std::memcpy(dst, src, std::min(piece, bytes));
  for (auto& t : th) t.join();
}

// A 2D block (rows x width bytes, device pitch = host pitch) of device
// memory -> pageable host, through the device's pinned double buffer: as
// many whole rows per staging block as fit, host threads scatter the rows.
sf_status staged_d2h_2d(int device, cudaStream_t cs, const char* dsrc, char* hdst, size_t pitch, size_t width,
                        size_t rows, unsigned threads);

// Host threads for the pinned -> pageable copies of one of `ndev` devices
// downloading at once.
unsigned copy_threads(size_t ndev) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return std::max(1u, std::min(16u, hw / static_cast<unsigned>(std::max<size_t>(1, ndev))));
}

// The device's two pinned staging slots (allocated on first use; false when
// no pinned memory is available). Caller holds S.mu.
bool ensure_staging(PinnedStaging& S) {
  constexpr size_t kSlot = 128ull << 20;
  if (S.slot[0]) return true;
  for (int i = 0; i < 2; ++i) {
    void* h = nullptr;
    if (cudaHostAlloc(&h, kSlot, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      if (S.slot[0]) cudaFreeHost(S.slot[0]);
      S.slot[0] = nullptr;
      return false;
    }
    S.slot[i] = static_cast<char*>(h);
  }
  S.bytes = kSlot;
  return true;
}

// dsrc (memory of `device`, the current device) -> hdst (pageable host), on cs.
sf_status staged_d2h(int device, cudaStream_t cs, const char* dsrc, char* hdst, size_t bytes, unsigned threads) {
  if (bytes == 0) return SF_OK;
  PinnedStaging& S = staging(device);
  std::lock_guard<std::mutex> lock(S.mu);
  if (!ensure_staging(S)) {  // no pinned memory to spare: the driver's own pageable path
    SF_CUDA(cudaMemcpyAsync(hdst, dsrc, bytes, cudaMemcpyDeviceToHost, cs));
    SF_CUDA(cudaStreamSynchronize(cs));
    return SF_OK;
  }
  cudaEvent_t ev[2];
  SF_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  if (cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess) {
    cudaEventDestroy(ev[0]);
    return fail(SF_ECUDA, "cudaEventCreate failed");
  }
  sf_status rc = SF_OK;
  const size_t nblk = (bytes + S.bytes - 1) / S.bytes;
  auto issue = [&](size_t b) -> sf_status {
    const size_t o = b * S.bytes;
    SF_CUDA(cudaMemcpyAsync(S.slot[b & 1], dsrc + o, std::min(S.bytes, bytes - o), cudaMemcpyDeviceToHost, cs));
    SF_CUDA(cudaEventRecord(ev[b & 1], cs));
    return SF_OK;
  };
  rc = issue(0);
  for (size_t b = 0; rc == SF_OK && b < nblk; ++b) {
    // slot (b+1)&1 was drained by block b-1's host copy, which has returned
    if (b + 1 < nblk) rc = issue(b + 1);
    if (rc != SF_OK) break;
    if (cudaEventSynchronize(ev[b & 1]) != cudaSuccess) {
      rc = fail(SF_ECUDA, std::string("staged download: ") + cudaGetErrorString(cudaGetLastError()));
      break;
    }
    const size_t o = b * S.bytes;
    parallel_memcpy(hdst + o, S.slot[b & 1], std::min(S.bytes, bytes - o), threads);
  }
  cudaStreamSynchronize(cs);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return rc;
}
// hsrc (pageable host) -> ddst (memory of `device`, the current device), on
// cs, through the device's pinned double buffer: host threads fill slot b+1
// while slot b's copy runs (pageable H2D goes through the driver's small
// staging buffers on one thread). Returns when the copy is done.
sf_status staged_h2d(int device, cudaStream_t cs, const char* hsrc, char* ddst, size_t bytes, unsigned threads) {
  if (bytes == 0) return SF_OK;
  PinnedStaging& S = staging(device);
  std::lock_guard<std::mutex> lock(S.mu);
  if (!ensure_staging(S)) {
    SF_CUDA(cudaMemcpyAsync(ddst, hsrc, bytes, cudaMemcpyHostToDevice, cs));
    SF_CUDA(cudaStreamSynchronize(cs));
    return SF_OK;
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } eg{ev};
  SF_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  SF_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const size_t nblk = (bytes + S.bytes - 1) / S.bytes;
  for (size_t b = 0; b < nblk; ++b) {
    const size_t o = b * S.bytes, len = std::min(S.bytes, bytes - o);
    if (b >= 2) SF_CUDA(cudaEventSynchronize(ev[b & 1]));  // slot b&1 was sent by block b-2
    parallel_memcpy(S.slot[b & 1], hsrc + o, len, threads);
    SF_CUDA(cudaMemcpyAsync(ddst + o, S.slot[b & 1], len, cudaMemcpyHostToDevice, cs));
    SF_CUDA(cudaEventRecord(ev[b & 1], cs));
  }
  SF_CUDA(cudaStreamSynchronize(cs));
  return SF_OK;
}

sf_status staged_d2h_2d(int device, cudaStream_t cs, const char* dsrc, char* hdst, size_t pitch, size_t width,
                        size_t rows, unsigned threads) {
  if (rows == 0 || width == 0) return SF_OK;
  if (width == pitch) return staged_d2h(device, cs, dsrc, hdst, width * rows, threads);
  PinnedStaging& S = staging(device);
  std::lock_guard<std::mutex> lock(S.mu);
  if (!ensure_staging(S)) {  // no pinned memory: the driver's own pageable 2D copy
    SF_CUDA(cudaMemcpy2DAsync(hdst, pitch, dsrc, pitch, width, rows, cudaMemcpyDeviceToHost, cs));
    SF_CUDA(cudaStreamSynchronize(cs));
    return SF_OK;
  }
  const size_t per = std::max<size_t>(1, S.bytes / width);  // rows per staging block
  const size_t nblk = (rows + per - 1) / per;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } eg{ev};
  SF_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  SF_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto issue = [&](size_t b) -> sf_status {
    const size_t r0 = b * per, nr = std::min(per, rows - r0);
    SF_CUDA(cudaMemcpy2DAsync(S.slot[b & 1], width, dsrc + r0 * pitch, pitch, width, nr, cudaMemcpyDeviceToHost, cs));
    SF_CUDA(cudaEventRecord(ev[b & 1], cs));
    return SF_OK;
  };
  SF_TRY(issue(0));
  for (size_t b = 0; b < nblk; ++b) {
    if (b + 1 < nblk) SF_TRY(issue(b + 1));
    SF_CUDA(cudaEventSynchronize(ev[b & 1]));
    const size_t r0 = b * per, nr = std::min(per, rows - r0);
    const char* src = S.slot[b & 1];
    // scatter the rows over host threads
    const size_t T = std::max<size_t>(1, std::min<size_t>(threads, nr));
    std::vector<std::thread> th;
    auto part = [&](size_t t) {
      for (size_t r = t; r < nr; r += T) std::memcpy(hdst + (r0 + r) * pitch, src + r * width, width);
    };
    for (size_t t = 1; t < T; ++t) th.emplace_back(part, t);
    part(0);
    for (auto& x : th) x.join();
  }
  return SF_OK;
}
}  // namespace

extern "C" {

const char* sf_last_error(void) { return sf::last_error(); }
const char* sf_version(void) { return "stripefrac-b200 0.1.0 (sm_100a)"; }

int32_t sf_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int i = 0; i < count; ++i) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, i) == cudaSuccess && prop.major == 10) ++ok;
  }
  return ok;
}

sf_status sf_trim_memory(int32_t device) {
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  std::vector<int> devs;
  SF_TRY(usable_devices(&ex, devs));
  if (cudaMemPool_t pool = device_pool(device)) {
    SF_CUDA(cudaSetDevice(device));
    SF_CUDA(cudaDeviceSynchronize());
    SF_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  return SF_OK;
}

sf_status sf_plan_create(const sf_problem* p, sf_metric metric, sf_precision prec, int32_t start,
                         int32_t stop, const sf_exec* ex, sf_plan** out) {
  if (!out) return fail(SF_EINVAL, "out is null");
  *out = nullptr;
  if (metric != SF_UNWEIGHTED && metric != SF_WEIGHTED_UNNORMALIZED && metric != SF_WEIGHTED_NORMALIZED &&
      metric != SF_GENERALIZED)
    return fail(SF_EINVAL, "unknown metric code " + std::to_string(static_cast<int>(metric)));
  const double alpha = ex ? ex->alpha : 0.0;
  if (metric == SF_GENERALIZED && !(std::isfinite(alpha) && alpha >= 0.0))
    return fail(SF_EINVAL, "generalized UniFrac needs a finite alpha >= 0");
  if (prec != SF_FP32 && prec != SF_FP64)
    return fail(SF_EINVAL, "unknown precision code " + std::to_string(static_cast<int>(prec)));
  const bool dbg = std::getenv("SF_DEBUG") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "stripefrac:   plan %s %.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tick).count());
    tick = now;
  };
  SF_TRY(validate_tree(p));
  // the single-chunk embedding schedule (every resident path; the chunked
  // dense paths rebuild it for their chunk size) reads only the tree: it is
  // built on a host thread while the table is validated, the devices are
  // set up, the table uploads and the fixed-point levels are formed
  Schedule sched_all;
  std::thread sched_thread([&] { sched_all = build_schedule(p, p->n_rows); });
  struct SchedJoiner {
    std::thread& t;
    ~SchedJoiner() {
      if (t.joinable()) t.join();
    }
  } sched_joiner{sched_thread};
  SF_TRY(validate_range(p->n_samples, start, stop));
  phase("validate tree");
  std::vector<int> devices;
  SF_TRY(usable_devices(ex, devices));
  phase("devices");

  auto plan = std::make_unique<sf_plan>();
  plan->metric = metric;
  plan->prec = prec;
  plan->n = p->n_samples;
  plan->E = p->n_rows;
  plan->start = start;
  plan->stop = stop;
  plan->bits = metric == SF_UNWEIGHTED;
  plan->exact = ex && (ex->flags & SF_EXEC_EXACT_NO_FMA);
  plan->mem_budget = (ex && ex->mem_budget_bytes > 0) ? static_cast<size_t>(ex->mem_budget_bytes) : 0;
  if (ex && ex->kernel != 0 && ex->kernel != 1 && ex->kernel != 2 && ex->kernel != 10 && ex->kernel != 11 &&
      ex->kernel != 12 && ex->kernel != 13)
    return fail(SF_EINVAL, "unknown kernel " + std::to_string(ex->kernel) +
                               " (1 dense, 2 sparse walk, 10 split, 11 weighted walk, 12 u-walk, 13 weighted split)");
  plan->kernel = (ex && ex->kernel >= 2) ? ex->kernel : 1;
  const int n = p->n_samples;
  // auto, unweighted: the intersection kernel (exact fixed-point sums), or
  // with SF_EXEC_EXACT_NO_FMA the sparse walk (the reference's adds in the
  // reference's order: bitwise identical); both keep every row resident, so
  // a budget too small for that selects the chunked dense kernel.
  if ((!ex || ex->kernel == 0) && metric == SF_UNWEIGHTED) {
    const int k = plan->exact ? 2 : 10;
    const bool fits = !(ex && ex->mem_budget_bytes > 0) ||
                      nodepacked_bytes(k, p->n_rows, n) <= static_cast<size_t>(ex->mem_budget_bytes);
    plan->kernel = fits ? k : 1;
  }
  // auto, weighted and generalized: the weighted split (kernel 13); in exact
  // mode the bitwise present-row walk (11)
  if ((!ex || ex->kernel == 0) && metric != SF_UNWEIGHTED) plan->kernel = plan->exact ? 11 : 13;
  if ((plan->kernel == 2 || plan->kernel == 10) && metric != SF_UNWEIGHTED)
    return fail(SF_EINVAL, "the sparse bit kernels implement the unweighted metric only");
  if (plan->kernel >= 11 && metric == SF_UNWEIGHTED)
    return fail(SF_EINVAL, "the weighted sparse walk implements the weighted metrics only");
  if (metric == SF_GENERALIZED && plan->kernel < 11)
    return fail(SF_EINVAL, "generalized UniFrac runs on the weighted kernels (11/12/13) only");
  plan->alpha = alpha;
  const bool wsp = plan->kernel == 11 || plan->kernel == 12 || plan->kernel == 13;
  const bool wuw = plan->kernel == 12 || plan->kernel == 13;
  if (plan->kernel == 13) {
    // light part's fixed-point grid: every sum (<= AL_k + AL_l <= 2 sum L, the
    // values being relative abundances <= 1) below 2^125, terms (<= 3 Lmax
    // 2^G in magnitude) in nd balanced 16-bit digits
    double tl = 0.0, lmax = 0.0;
    for (int32_t r = 0; r < p->n_rows; ++r) {
      tl += p->lengths[r];
      lmax = std::max(lmax, p->lengths[r]);
    }
    // generalized: a shared row's terms reach (u + v)^alpha L <= 2^alpha L
    const double f = metric == SF_GENERALIZED ? std::max(1.0, std::exp2(alpha)) : 1.0;
    const double bound = (2.0 * tl + 4.0 * lmax) * f + 1.0;
    plan->ws_G = 125 - (std::ilogb(bound) + 1);
    const int term_bits = (lmax > 0 ? std::ilogb(3.0 * lmax * f) + 2 : 1) + plan->ws_G + 1;
    plan->ws_nd = std::min(8, std::max(4, (term_bits + 15) / 16));
  }
  {
    const char* de = std::getenv("SF_WS_DENSE_EMBED");
    plan->wbits = plan->kernel == 13 && !(de && std::atoi(de) == 1);
  }
  plan->row_words = (plan->bits || plan->wbits) ? (n + 31) / 32 : ((n + 1) / 2) * 2;
  const size_t w = prec == SF_FP64 ? 8 : 4;
  const bool has_t = metric != SF_WEIGHTED_UNNORMALIZED;

  // stripe split: the reference's worker split formula (kernels.hpp:302-303)
  const int G = static_cast<int>(devices.size());
  const int span = stop - start;
  if (G > span) devices.resize(static_cast<size_t>(span));
  const int Gu = static_cast<int>(devices.size());
  for (int g = 0; g < Gu; ++g) {
    auto d = std::make_unique<DeviceState>();
    d->dev = devices[static_cast<size_t>(g)];
    d->a = start + static_cast<int>(static_cast<int64_t>(span) * g / Gu);
    d->b = start + static_cast<int>(static_cast<int64_t>(span) * (g + 1) / Gu);
    plan->devs.push_back(std::move(d));
  }

  // the table upload (C3: 192 MB from pageable memory) runs on a host thread
  // while this one validates the table and sizes the plan (a table that
  // fails validation is uploaded for nothing: the error is returned after
  // the join)
  std::vector<sf_status> up_status(plan->devs.size(), SF_OK);
  std::vector<std::string> up_error(plan->devs.size());
  std::thread uploader([&] {
    for (size_t i = 0; i < plan->devs.size(); ++i) {
      DeviceState& d = *plan->devs[i];
      auto run = [&]() -> sf_status {
        SF_CUDA(cudaSetDevice(d.dev));
        SF_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
        const int64_t F = p->n_features;
        const int64_t nnz = p->feat_ptr[F];
        SF_TRY(upload(d.lens, d.dev, p->lengths, static_cast<size_t>(plan->E), d.stream, "lengths"));
        SF_TRY(upload(d.feat_ptr, d.dev, p->feat_ptr, static_cast<size_t>(F + 1), d.stream, "feat_ptr"));
        // the table's big arrays (C3: 180 MB) through the pinned staging buffers
        SF_TRY(d.sidx.alloc(d.dev, static_cast<size_t>(nnz) * 4, "sample_idx"));
        SF_TRY(d.counts.alloc(d.dev, static_cast<size_t>(nnz) * 8, "counts"));
        const unsigned th = copy_threads(plan->devs.size());
        if (host_pinned(p->sample_idx))
          SF_CUDA(cudaMemcpyAsync(d.sidx.p, p->sample_idx, static_cast<size_t>(nnz) * 4, cudaMemcpyHostToDevice, d.stream));
        else
          SF_TRY(staged_h2d(d.dev, d.stream, reinterpret_cast<const char*>(p->sample_idx), d.sidx.as<char>(),
                            static_cast<size_t>(nnz) * 4, th));
        if (host_pinned(p->counts))
          SF_CUDA(cudaMemcpyAsync(d.counts.p, p->counts, static_cast<size_t>(nnz) * 8, cudaMemcpyHostToDevice, d.stream));
        else
          SF_TRY(staged_h2d(d.dev, d.stream, reinterpret_cast<const char*>(p->counts), d.counts.as<char>(),
                            static_cast<size_t>(nnz) * 8, th));
        SF_TRY(upload(d.totals, d.dev, p->sample_totals, static_cast<size_t>(n), d.stream, "totals"));
        return SF_OK;
      };
      up_status[i] = run();
      if (up_status[i] != SF_OK) {
        up_error[i] = sf::last_error();
        return;
      }
    }
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{uploader};
  phase("spawn uploader");
  SF_TRY(validate_table(p));
  phase("validate table");

  // chunk capacity from the smallest device budget
  const size_t row_bytes = static_cast<size_t>(plan->row_words) * ((plan->bits || plan->wbits) ? 4 : 8);
  // kernel 11 holds, per chunk row, the dense row + its share of the value
  // pool (worst case n values) + presence words / counts / offsets
  const size_t wsp_row_bytes =
      wsp ? (wuw ? 0 : static_cast<size_t>(n) * w) + (static_cast<size_t>(sparse_n_ext(n)) * 12 + 31) / 32 : 0;
  // kernel 12 keeps the whole problem's presence words, offsets and values
  const uint64_t pbound = wuw ? present_bound(p) : 0;
  if (wuw && pbound >= (1ull << 32))
    return fail(SF_EINVAL, "weighted u-walk: more than 2^32 present entries; use kernel 11");
  const size_t wuw_fixed =
      wuw ? static_cast<size_t>((plan->E + 31) / 32) * static_cast<size_t>(sparse_n_ext(n)) * 8 +
                static_cast<size_t>(pbound) * w * (metric == SF_GENERALIZED ? 2 : 1)
          : 0;
  size_t budget = SIZE_MAX;
  // the resident sparse bit kernels (2-10) take every row in one chunk
  // whatever the budget, so they skip the free-memory query here (it took
  // 28-64 ms on some calls); kernel 10 sizes its light pass at device setup
  const bool budget_free = (plan->kernel >= 2 && !wsp) || plan->wbits;
  for (auto& d : plan->devs) {
    if (budget_free) break;
    SF_CUDA(cudaSetDevice(d->dev));
    const size_t stripes_b = static_cast<size_t>(d->b - d->a) * n * w * (has_t ? 2 : 1);
    const size_t csr_b = static_cast<size_t>(p->feat_ptr[p->n_features]) * 12 + static_cast<size_t>(plan->E) * 64;
    const size_t fixed_b = stripes_b + csr_b + wuw_fixed + (512ull << 20);
    if (!(ex && ex->mem_budget_bytes > 0)) {
      // one chunk of every row (no pending rows) if a probe allocation of
      // it plus the fixed part (with the 4/3 margin below) succeeds; the
      // memory returns to the pool. cudaMemGetInfo stalls up to ~100 ms.
      const size_t whole = static_cast<size_t>(plan->E) * (row_bytes + wsp_row_bytes);
      if (whole / 3 < (SIZE_MAX - fixed_b) / 4 &&
          probe_fits(d->dev, fixed_b + whole + whole / 3, fixed_b - (512ull << 20) + whole)) {
        budget = std::min(budget, whole);
        continue;
      }
    }
    size_t freeb = 0;
    SF_TRY(device_free_bytes(d->dev, &freeb));
    const size_t avail = freeb > fixed_b ? freeb - fixed_b : 0;
    budget = std::min(budget, avail * 3 / 4);
  }
  if (ex && ex->mem_budget_bytes > 0) budget = std::min(budget, static_cast<size_t>(ex->mem_budget_bytes));
  phase("budget");

  int64_t cmax = static_cast<int64_t>(budget / std::max<size_t>(row_bytes + wsp_row_bytes, 1));
  if (plan->kernel >= 2 && !wsp) cmax = plan->E;  // the sparse bit paths keep all rows
  if (wsp) {
    // 32-row words never straddle chunks; uint32 pool offsets
    cmax = std::min<int64_t>(cmax, static_cast<int64_t>(UINT32_MAX / static_cast<uint64_t>(n)) / 32 * 32);
    if (cmax < plan->E) cmax = cmax / 32 * 32;
    if (cmax < 32) cmax = std::min<int64_t>(32, plan->E);
  }
  if (plan->wbits) cmax = plan->E;  // bit rows: every row in one chunk
  cmax = std::min<int64_t>(cmax, plan->E);
  if (cmax < 1) return fail(SF_ENOMEM, "not enough device memory for one embedding row");
  FixedLevels fl;
  if (plan->kernel == 10) {
    SF_TRY(fixed_levels(p->lengths, plan->E, prec == SF_FP32, fl));
    phase("fixed-point levels");
  }
  sched_thread.join();
  phase("schedule (overlapped)");
  for (;;) {
    if (cmax == plan->E && sched_all.cmax == cmax)
      plan->sched = std::move(sched_all);
    else
      plan->sched = build_schedule(p, static_cast<int32_t>(cmax));
    const size_t need = (static_cast<size_t>(cmax) + static_cast<size_t>(plan->sched.n_pending)) * row_bytes +
                        static_cast<size_t>(cmax) * wsp_row_bytes;
    if (need <= budget || cmax == 1 || (plan->kernel >= 2 && !wsp) || (wsp && cmax <= 32) || plan->wbits) break;
    cmax = std::max<int64_t>(1, cmax * 3 / 4);
    if (wsp) cmax = std::max<int64_t>(32, cmax / 32 * 32);
  }
  plan->stats.n_chunks = plan->sched.chunks.size();

  uploader.join();
  for (size_t i = 0; i < up_status.size(); ++i)
    if (up_status[i] != SF_OK) return fail(up_status[i], up_error[i]);
  phase("upload table (overlapped)");
  if (plan->kernel == 10) {
    plan->scale = fl.scale;
    plan->lo_bits = fl.lo_bits;
    plan->vb = fl.vb;
    plan->levels = fl.levels;
    plan->fix = std::move(fl.fix);
    plan->deep_rows = std::move(fl.deep_rows);
    plan->dfix = std::move(fl.dfix);
  }
  for (auto& dp : plan->devs) {
    DeviceState& d = *dp;
    SF_CUDA(cudaSetDevice(d.dev));
    const size_t slots = static_cast<size_t>(d.b - d.a) * static_cast<size_t>(n);
    SF_TRY(d.dist.alloc(d.dev, slots * w, "distances"));
    if (has_t) SF_TRY(d.tot.alloc(d.dev, slots * w, "totals"));
    SF_TRY(d.exec_ctr.alloc(d.dev, 2 * sizeof(unsigned long long), "counters"));
    if (wsp) {
      SF_TRY(upload_schedule(d, plan->sched));
      const int32_t cm = plan->sched.cmax;
      SF_TRY(d.emb.alloc(d.dev, static_cast<size_t>(cm) * row_bytes, "embedding chunk"));
      SF_TRY(d.pend.alloc(d.dev, static_cast<size_t>(std::max(plan->sched.n_pending, 1)) * row_bytes,
                          "pending rows"));
      const int64_t cells = static_cast<int64_t>((cm + 31) / 32) * sparse_n_ext(n);
      SF_TRY(d.wnb.alloc(d.dev, static_cast<size_t>(cells) * 4, "presence words"));
      SF_TRY(d.wcnt.alloc(d.dev, static_cast<size_t>(cells) * 4, "presence counts"));
      SF_TRY(d.woff.alloc(d.dev, static_cast<size_t>(cells) * 4, "pool offsets"));
      if (wuw) {
        const int64_t gcells = static_cast<int64_t>((plan->E + 31) / 32) * sparse_n_ext(n);
        SF_TRY(d.wnb.alloc(d.dev, static_cast<size_t>(gcells) * 4, "presence words"));
        SF_TRY(d.woff.alloc(d.dev, static_cast<size_t>(gcells) * 4, "pool offsets"));
        SF_TRY(d.wpool.alloc(d.dev, static_cast<size_t>(pbound) * w, "value pool"));
        if (metric == SF_GENERALIZED)
          SF_TRY(d.wpoola.alloc(d.dev, static_cast<size_t>(pbound) * w, "generalized pool"));
        SF_TRY(d.wA.alloc(d.dev, static_cast<size_t>(n) * 16, "column sums"));
        SF_TRY(d.nzmask.alloc(d.dev, static_cast<size_t>(((plan->E + 31) / 32 + 31) / 32) * static_cast<size_t>(n) * 4,
                              "nonzero-word masks"));
        SF_TRY(d.wbase.alloc(d.dev, 16, "pool base"));
        SF_TRY(sparse_prepare_lens(plan.get(), d, p));
      } else {
        SF_TRY(d.wpool.alloc(d.dev, static_cast<size_t>(cm) * static_cast<size_t>(n) * w, "value pool"));
      }
      size_t tmp = 0;
      SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d.wcnt.as<uint32_t>(), d.woff.as<uint32_t>(),
                                            static_cast<int>(cells), d.stream));
      d.cub_bytes = tmp;
      SF_TRY(d.cubtmp.alloc(d.dev, tmp, "scan scratch"));
    } else if (plan->kernel >= 2) {
      SF_TRY(upload_schedule(d, plan->sched));
      SF_TRY(d.emb.alloc(d.dev, static_cast<size_t>(plan->E) * row_bytes, "embedding rows"));
      SF_TRY(d.pend.alloc(d.dev, 16, "pending rows"));
      if (plan->kernel == 10) {
        phase("device alloc");
        SF_TRY(split_prepare(plan.get(), d));
        phase("node-packed prepare");
        {
          const int span = d.b - d.a;
          const size_t after = static_cast<size_t>(plan->E) * 4 * (3 + 2 * static_cast<size_t>(split_heavy_min(n)));
          const char* lm0 = std::getenv("SF_LIGHT_MODE");
          d.light_lazy = light_banded() && !(lm0 && std::string(lm0) == "band") && heavy_gemm_enabled() &&
                         static_cast<uint64_t>(plan->E) * static_cast<uint64_t>(split_heavy_min(n)) < (1ull << 32) &&
                         split_heavy_min(n) <= 65535;
          d.light_sized = false;
          if (d.light_lazy)
            d.light_pass = span;  // placeholder: sized in run_device after the GEMM operands
          else
            SF_TRY(light_sums_alloc(plan.get(), d, after));
          SF_TRY(d.mcount.alloc(d.dev, static_cast<size_t>(plan->E) * 4, "row presence counts"));
          // u32 member offsets; u16 cursors (light rows have < heavy_min members)
          d.banded = light_banded() &&
                     static_cast<uint64_t>(plan->E) * static_cast<uint64_t>(split_heavy_min(n)) < (1ull << 32) &&
                     split_heavy_min(n) <= 65535;
          if (d.banded) {
            const size_t E1 = static_cast<size_t>(plan->E) + 1;
            SF_TRY(d.lcnt.alloc(d.dev, E1 * 4, "light member counts"));
            SF_TRY(d.lptr.alloc(d.dev, E1 * 4, "light member offsets"));
            // light rows have |X_e| < heavy_min members
            SF_TRY(d.lmem.alloc(d.dev, static_cast<size_t>(plan->E) * static_cast<size_t>(split_heavy_min(n)) * 4,
                                "light members"));
            SF_TRY(d.lcur.alloc(d.dev, static_cast<size_t>(plan->E) * static_cast<size_t>(split_heavy_min(n)) * 4,
                                "light member cursors"));
            size_t tmp = 0;
            SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d.lcnt.as<uint32_t>(), d.lptr.as<uint32_t>(),
                                                  static_cast<int>(E1), d.stream));
            d.lscan_bytes = tmp;
            SF_TRY(d.lscantmp.alloc(d.dev, tmp, "light scan scratch"));
            // column-owned light scatter (default; SF_LIGHT_MODE=band: the banded kernel)
            const char* lm = std::getenv("SF_LIGHT_MODE");
            d.light_columns = !(lm && std::string(lm) == "band");
            if (d.light_columns) {
              SF_TRY(d.ccnt.alloc(d.dev, static_cast<size_t>(n + 1) * 4, "column entry counts"));
              SF_TRY(d.cptr.alloc(d.dev, static_cast<size_t>(n + 1) * 4, "column entry offsets"));
              size_t ct = 0;
              SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, ct, d.ccnt.as<uint32_t>(), d.cptr.as<uint32_t>(), n + 1,
                                                    d.stream));
              d.cscan_bytes = ct;
              SF_TRY(d.cscantmp.alloc(d.dev, ct, "column scan scratch"));
            }
          }
        }
      } else {
        SF_TRY(sparse_prepare(plan.get(), d, p));
      }
    } else {
      SF_TRY(upload_schedule(d, plan->sched));
      SF_TRY(d.emb.alloc(d.dev, static_cast<size_t>(cmax) * row_bytes, "embedding chunk"));
      SF_TRY(d.pend.alloc(d.dev, static_cast<size_t>(std::max(plan->sched.n_pending, 1)) * row_bytes,
                          "pending rows"));
    }
  }
  phase("device setup");
  *out = plan.release();
  return SF_OK;
}

sf_status sf_plan_run(sf_plan* plan, int32_t finalize) {
  if (!plan) return fail(SF_EINVAL, "plan is null");
  for (auto& d : plan->devs) d->launches = 0;
  SF_TRY(for_each_device(plan, [&](DeviceState& d) { return run_device(plan, d, finalize); }));
  plan->ran = true;
  plan->finalized = finalize != 0;
  return SF_OK;
}

sf_status sf_plan_sync(sf_plan* plan) {
  if (!plan) return fail(SF_EINVAL, "plan is null");
  double emb = 0, str = 0, fin = 0, tot = 0, tens = 0;
  uint64_t exec = 0, fpops = 0, tops = 0;
  for (auto& dp : plan->devs) {
    DeviceState& d = *dp;
    SF_CUDA(cudaSetDevice(d.dev));
    SF_CUDA(cudaStreamSynchronize(d.stream));
    if (d.copy_stream) SF_CUDA(cudaStreamSynchronize(d.copy_stream));
    if (!plan->ran) continue;
    double e_ms = 0, s_ms = 0, f_ms = 0, t_ms = 0;
    const size_t ne = d.events.size();
    for (size_t ci = 0; ci < plan->sched.chunks.size(); ++ci) {
      float a = 0, b = 0;
      SF_CUDA(cudaEventElapsedTime(&a, d.events[1 + 3 * ci], d.events[2 + 3 * ci]));
      SF_CUDA(cudaEventElapsedTime(&b, d.events[2 + 3 * ci], d.events[3 + 3 * ci]));
      e_ms += a;
      s_ms += b;
    }
    float f = 0, t = 0;
    SF_CUDA(cudaEventElapsedTime(&f, d.events[ne - 2], d.events[ne - 1]));
    SF_CUDA(cudaEventElapsedTime(&t, d.events[0], d.events[ne - 1]));
    f_ms = f;
    t_ms = t;
    double g_ms = 0;
    for (size_t i = 0; i < d.gemm_count; ++i) {
      float g = 0;
      SF_CUDA(cudaEventElapsedTime(&g, d.gemm_ev[2 * i], d.gemm_ev[2 * i + 1]));
      g_ms += g;
    }
    tens = std::max(tens, g_ms);
    tops += d.gemm_ops;
    exec += d.heavy_updates;
    emb = std::max(emb, e_ms);
    str = std::max(str, s_ms);
    fin = std::max(fin, f_ms);
    tot = std::max(tot, t_ms);
    unsigned long long c[2] = {0, 0};
    SF_CUDA(cudaMemcpy(c, d.exec_ctr.p, sizeof(c), cudaMemcpyDeviceToHost));
    exec += c[0];
    fpops += c[1] + d.host_fp64_ops;
  }
  plan->stats.launches = 0;
  for (auto& dp : plan->devs) plan->stats.launches += dp->launches;
  plan->stats.embed_ms = emb;
  plan->stats.stripe_ms = str;
  plan->stats.finalize_ms = fin;
  plan->stats.total_ms = tot;
  plan->stats.updates_exec = exec;
  plan->stats.fp64_ops = fpops;
  plan->stats.tensor_ops = tops;
  plan->stats.tensor_ms = tens;
  plan->stats.updates_alg = static_cast<uint64_t>(plan->E) * static_cast<uint64_t>(plan->stop - plan->start) *
                            static_cast<uint64_t>(plan->n);
  return SF_OK;
}



sf_status sf_plan_download(sf_plan* plan, void* dist_out, void* tot_out) {
  if (!plan) return fail(SF_EINVAL, "plan is null");
  if (!plan->ran) return fail(SF_ESTATE, "plan has not run");
  if (!dist_out) return fail(SF_EINVAL, "dist_out is null");
  const bool has_t = plan->metric != SF_WEIGHTED_UNNORMALIZED;
  const size_t w = plan->prec == SF_FP64 ? 8 : 4;
  const bool pageable_d = !host_pinned(dist_out);
  const bool pageable_t = tot_out && !host_pinned(tot_out);
  const unsigned threads = copy_threads(plan->devs.size());
  return for_each_device(plan, [&](DeviceState& d) -> sf_status {
    SF_CUDA(cudaSetDevice(d.dev));
    const size_t off = static_cast<size_t>(d.a - plan->start) * plan->n * w;
    const size_t bytes = static_cast<size_t>(d.b - d.a) * plan->n * w;
    if (pageable_d) {
      SF_CUDA(cudaStreamSynchronize(d.stream));
      SF_TRY(staged_d2h(d.dev, d.stream, d.dist.as<char>(), static_cast<char*>(dist_out) + off, bytes, threads));
    } else {
      SF_CUDA(cudaMemcpyAsync(static_cast<char*>(dist_out) + off, d.dist.p, bytes, cudaMemcpyDeviceToHost, d.stream));
    }
    if (has_t && tot_out) {
      if (pageable_t) {
        SF_CUDA(cudaStreamSynchronize(d.stream));
        SF_TRY(staged_d2h(d.dev, d.stream, d.tot.as<char>(), static_cast<char*>(tot_out) + off, bytes, threads));
      } else {
        SF_CUDA(cudaMemcpyAsync(static_cast<char*>(tot_out) + off, d.tot.p, bytes, cudaMemcpyDeviceToHost, d.stream));
      }
    }
    SF_CUDA(cudaStreamSynchronize(d.stream));
    return SF_OK;
  });
}

sf_status sf_plan_stats(const sf_plan* plan, sf_stats* out) {
  if (!plan || !out) return fail(SF_EINVAL, "null argument");
  *out = plan->stats;
  return SF_OK;
}

void sf_plan_destroy(sf_plan* plan) { delete plan; }

sf_status sf_compute_stripes(const sf_problem* p, sf_metric metric, sf_precision prec,
                             int32_t start, int32_t stop, void* dist_out, void* tot_out,
                             int32_t finalize, const sf_exec* ex, sf_stats* stats_out) {
  if (!dist_out) return fail(SF_EINVAL, "dist_out is null");
  if (metric != SF_WEIGHTED_UNNORMALIZED && !tot_out)
    return fail(SF_EINVAL, "tot_out is required for ratio metrics");
  sf_plan* plan = nullptr;
  const bool dbg = std::getenv("SF_DEBUG") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  SF_TRY(sf_plan_create(p, metric, prec, start, stop, ex, &plan));
  std::unique_ptr<sf_plan> guard(plan);
  if (dbg)
    std::fprintf(stderr, "stripefrac: plan_create %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  const bool all_pinned = host_pinned(dist_out) && (!tot_out || host_pinned(tot_out));
  if (plan->kernel == 10) {
    // the split kernel computes the stripes in chunks; each finished chunk is
    // copied while the later chunks compute: pinned destinations straight
    // from a copy stream, pageable ones staged through the device's pinned
    // double buffer by host threads. One host thread per device.
    const size_t w = prec == SF_FP64 ? 8 : 4;
    const unsigned threads = copy_threads(plan->devs.size());
    for (auto& d : plan->devs) d->launches = 0;
    SF_TRY(for_each_device(plan, [&](DeviceState& d) -> sf_status {
      SF_CUDA(cudaSetDevice(d.dev));
      const size_t off = static_cast<size_t>(d.a - plan->start) * plan->n * w;
      char* hd = static_cast<char*>(dist_out) + off;
      char* ht = tot_out ? static_cast<char*>(tot_out) + off : nullptr;
      d.chunk_spans.clear();
      d.defer_copy = !all_pinned;
      const sf_status rc = run_device(plan, d, finalize, hd, ht);
      d.defer_copy = false;
      SF_TRY(rc);
      const size_t pitch = static_cast<size_t>(plan->n) * w;
      for (size_t ci = 0; ci < d.chunk_spans.size(); ++ci) {
        SF_CUDA(cudaEventSynchronize(d.chunk_events[ci]));
        const DeviceState::Span& sp = d.chunk_spans[ci];
        const size_t co = static_cast<size_t>(sp.row0) * pitch + static_cast<size_t>(sp.col0) * w;
        const size_t width = static_cast<size_t>(sp.cols) * w, rows = static_cast<size_t>(sp.rows);
        SF_TRY(staged_d2h_2d(d.dev, d.copy_stream, d.dist.as<char>() + co, hd + co, pitch, width, rows, threads));
        if (ht && metric != SF_WEIGHTED_UNNORMALIZED)
          SF_TRY(staged_d2h_2d(d.dev, d.copy_stream, d.tot.as<char>() + co, ht + co, pitch, width, rows, threads));
      }
      return SF_OK;
    }));
    plan->ran = true;
    plan->finalized = finalize != 0;
    SF_TRY(sf_plan_sync(plan));
  } else {
    SF_TRY(sf_plan_run(plan, finalize));
    SF_TRY(sf_plan_sync(plan));
    SF_TRY(sf_plan_download(plan, dist_out, tot_out));
  }
  if (dbg)
    std::fprintf(stderr, "stripefrac: compute_stripes %.1f ms (device %.1f ms)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                 plan->stats.total_ms);
  if (stats_out) *stats_out = plan->stats;
  return SF_OK;
}

sf_status sf_accumulate_batch(const void* emb, const void* lengths, int32_t filled,
                              int32_t n_samples, int32_t padded, sf_metric metric,
                              sf_precision prec, int32_t start, int32_t stop, void* dist_inout,
                              void* tot_inout, int32_t device) {
  if (filled < 1) return fail(SF_EINVAL, "embedding batch is empty");
  if (n_samples < 2) return fail(SF_EINVAL, "need at least 2 samples");
  if (padded < n_samples) return fail(SF_EINVAL, "embedding batch shape is inconsistent");
  if (!emb || !lengths || !dist_inout) return fail(SF_EINVAL, "null argument");
  if (metric != SF_UNWEIGHTED && metric != SF_WEIGHTED_UNNORMALIZED && metric != SF_WEIGHTED_NORMALIZED)
    return fail(SF_EINVAL, "unknown metric code " + std::to_string(static_cast<int>(metric)));
  const bool has_t = metric != SF_WEIGHTED_UNNORMALIZED;
  if (has_t && !tot_inout) return fail(SF_EINVAL, "tot_inout is required for ratio metrics");
  if (prec != SF_FP32 && prec != SF_FP64) return fail(SF_EINVAL, "unknown precision");
  SF_TRY(validate_range(n_samples, start, stop));
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  std::vector<int> devs;
  SF_TRY(usable_devices(&ex, devs));
  SF_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  SF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  const size_t w = prec == SF_FP64 ? 8 : 4;
  DevBuf demb, dlen, ddist, dtot;
  std::vector<double> lens(static_cast<size_t>(filled));
  for (int i = 0; i < filled; ++i)
    lens[static_cast<size_t>(i)] = prec == SF_FP64 ? static_cast<const double*>(lengths)[i]
                                                   : static_cast<double>(static_cast<const float*>(lengths)[i]);
  SF_TRY(demb.alloc(device, static_cast<size_t>(filled) * padded * w, "batch"));
  SF_CUDA(cudaMemcpyAsync(demb.p, emb, static_cast<size_t>(filled) * padded * w, cudaMemcpyHostToDevice, st));
  SF_TRY(upload(dlen, device, lens.data(), lens.size(), st, "lengths"));
  const size_t slots = static_cast<size_t>(stop - start) * n_samples;
  SF_TRY(ddist.alloc(device, slots * w, "distances"));
  SF_CUDA(cudaMemcpyAsync(ddist.p, dist_inout, slots * w, cudaMemcpyHostToDevice, st));
  if (has_t) {
    SF_TRY(dtot.alloc(device, slots * w, "totals"));
    SF_CUDA(cudaMemcpyAsync(dtot.p, tot_inout, slots * w, cudaMemcpyHostToDevice, st));
  }
  StripeArgs a;
  a.emb = demb.p;
  a.row_stride = padded;
  a.lens = dlen.as<double>();
  a.C = filled;
  a.n = n_samples;
  a.s_begin = start;
  a.s_end = stop;
  a.dist = ddist.p;
  a.tot = has_t ? dtot.p : nullptr;
  a.exec_updates = nullptr;
  SF_TRY(launch_stripes(metric, prec, prec == SF_FP64 ? kSrcF64 : kSrcF32, false, a, st));
  SF_CUDA(cudaMemcpyAsync(dist_inout, ddist.p, slots * w, cudaMemcpyDeviceToHost, st));
  if (has_t) SF_CUDA(cudaMemcpyAsync(tot_inout, dtot.p, slots * w, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  return SF_OK;
}

sf_status sf_embed_rows(const sf_problem* p, int32_t weighted, int32_t r0, int32_t r1,
                        double* out, int32_t padded, int32_t device) {
  SF_TRY(validate_problem(p));
  if (r0 < 0 || r1 > p->n_rows || r0 > r1) return fail(SF_EINVAL, "row range out of bounds");
  if (padded < p->n_samples) return fail(SF_EINVAL, "padded width is smaller than the sample count");
  if (!out && r1 > r0) return fail(SF_EINVAL, "out is null");
  if (r1 == r0) return SF_OK;
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  // an embed-only plan: one stripe, one chunk holding every row
  sf_plan* raw = nullptr;
  const sf_metric m = weighted ? SF_WEIGHTED_UNNORMALIZED : SF_UNWEIGHTED;
  ex.mem_budget_bytes = 0;
  ex.kernel = weighted ? 12 : 0;  // dense value rows (kernel 13 keeps presence bits only)
  SF_TRY(sf_plan_create(p, m, SF_FP64, 0, 1, &ex, &raw));
  std::unique_ptr<sf_plan> plan(raw);
  if (plan->sched.chunks.size() != 1)
    return fail(SF_ENOMEM, "sf_embed_rows needs the whole embedding to fit on the device");
  DeviceState& d = *plan->devs[0];
  SF_TRY(run_device(plan.get(), d, 0));
  SF_CUDA(cudaStreamSynchronize(d.stream));
  const int n = p->n_samples;
  const int64_t rw = plan->row_words;
  const int64_t rows = r1 - r0;
  if (plan->bits) {
    std::vector<uint32_t> h(static_cast<size_t>(rows * rw));
    SF_CUDA(cudaMemcpy(h.data(), d.emb.as<uint32_t>() + r0 * rw, h.size() * 4, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < rows; ++r)
      for (int c = 0; c < padded; ++c)
        out[r * padded + c] = c < n ? static_cast<double>((h[static_cast<size_t>(r * rw + (c >> 5))] >> (c & 31)) & 1u) : 0.0;
  } else {
    std::vector<double> h(static_cast<size_t>(rows * rw));
    SF_CUDA(cudaMemcpy(h.data(), d.emb.as<double>() + r0 * rw, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < rows; ++r)
      for (int c = 0; c < padded; ++c) out[r * padded + c] = c < n ? h[static_cast<size_t>(r * rw + c)] : 0.0;
  }
  return SF_OK;
}

sf_status sf_finalize(sf_precision prec, int64_t count, void* dist_inout, const void* tot,
                      int32_t device) {
  if (count < 0 || (count > 0 && (!dist_inout || !tot))) return fail(SF_EINVAL, "bad arguments");
  if (prec != SF_FP32 && prec != SF_FP64) return fail(SF_EINVAL, "unknown precision");
  if (count == 0) return SF_OK;
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  std::vector<int> devs;
  SF_TRY(usable_devices(&ex, devs));
  SF_CUDA(cudaSetDevice(device));
  const size_t w = prec == SF_FP64 ? 8 : 4;
  DevBuf dd, dt;
  SF_TRY(dd.alloc(device, static_cast<size_t>(count) * w, "distances"));
  SF_TRY(dt.alloc(device, static_cast<size_t>(count) * w, "totals"));
  SF_CUDA(cudaMemcpy(dd.p, dist_inout, static_cast<size_t>(count) * w, cudaMemcpyHostToDevice));
  SF_CUDA(cudaMemcpy(dt.p, tot, static_cast<size_t>(count) * w, cudaMemcpyHostToDevice));
  const int blocks = grid_for(count, 256);
  if (prec == SF_FP64)
    finalize_kernel<double><<<blocks, 256>>>(dd.as<double>(), dt.as<double>(), count);
  else
    finalize_kernel<float><<<blocks, 256>>>(dd.as<float>(), dt.as<float>(), count);
  SF_CUDA(cudaGetLastError());
  SF_CUDA(cudaMemcpy(dist_inout, dd.p, static_cast<size_t>(count) * w, cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_condense(sf_precision prec, int32_t n, int32_t start, int32_t stop, const void* dist,
                      double* out, int32_t device) {
  if (!dist || !out) return fail(SF_EINVAL, "null argument");
  if (prec != SF_FP32 && prec != SF_FP64) return fail(SF_EINVAL, "unknown precision");
  if (n < 2) return fail(SF_EINVAL, "need at least 2 samples");
  SF_TRY(validate_range(n, start, stop));
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  std::vector<int> devs;
  SF_TRY(usable_devices(&ex, devs));
  SF_CUDA(cudaSetDevice(device));
  const size_t w = prec == SF_FP64 ? 8 : 4;
  const size_t slots = static_cast<size_t>(stop - start) * n;
  const size_t nn = static_cast<size_t>(n) * n;
  DevBuf dd, dout, dbad;
  SF_TRY(dd.alloc(device, slots * w, "stripes"));
  SF_TRY(dout.alloc(device, nn * 8, "matrix"));
  SF_TRY(dbad.alloc(device, sizeof(int), "flag"));
  SF_CUDA(cudaMemcpy(dd.p, dist, slots * w, cudaMemcpyHostToDevice));
  SF_CUDA(cudaMemcpy(dout.p, out, nn * 8, cudaMemcpyHostToDevice));
  SF_CUDA(cudaMemset(dbad.p, 0, sizeof(int)));
  const int blocks = grid_for(static_cast<int64_t>(slots), 256);
  if (prec == SF_FP64)
    condense_kernel<double><<<blocks, 256>>>(dd.as<double>(), n, start, stop, dout.as<double>(), dbad.as<int>());
  else
    condense_kernel<float><<<blocks, 256>>>(dd.as<float>(), n, start, stop, dout.as<double>(), dbad.as<int>());
  SF_CUDA(cudaGetLastError());
  int bad = 0;
  SF_CUDA(cudaMemcpy(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) return fail(SF_EINVAL, "condense: duplicated slot disagrees");
  SF_CUDA(cudaMemcpy(out, dout.p, nn * 8, cudaMemcpyDeviceToHost));
  return SF_OK;
}

// ---------------------------------------------------------------- condense
// condense (stripes.cpp:68-129) of a finalized full-range plan, on device:
// every device's stripe block is condensed into one n x n fp64 matrix on the
// plan's first device (other devices' blocks cross NVLink with a peer copy),
// the diagonal is zeroed, the even-n duplicate copies are verified, and the
// matrix is copied once into the caller's row-major n x n buffer (pinned:
// one async copy; pageable: staged through the device's pinned double buffer).
sf_status sf_plan_condense(sf_plan* plan, double* out) {
  if (!plan || !out) return fail(SF_EINVAL, "null argument");
  if (!plan->ran) return fail(SF_ESTATE, "plan has not run");
  if (!plan->finalized) return fail(SF_EINVAL, "condense needs finalized stripes");
  const int n = plan->n;
  if (plan->start != 0 || plan->stop != n / 2)
    return fail(SF_EINVAL, "stripe parts do not tile [0, " + std::to_string(n / 2) + ")");
  SF_TRY(sf_plan_sync(plan));
  DeviceState& d0 = *plan->devs.front();
  SF_CUDA(cudaSetDevice(d0.dev));
  const cudaStream_t st = d0.stream;
  const size_t w = plan->prec == SF_FP64 ? 8 : 4;
  const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);
  DevBuf mat, bad, peer;
  SF_TRY(mat.alloc(d0.dev, nn * 8, "distance matrix"));
  SF_TRY(bad.alloc(d0.dev, sizeof(int), "condense flag"));
  SF_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  for (auto& dp : plan->devs) {
    const DeviceState& d = *dp;
    const size_t slots = static_cast<size_t>(d.b - d.a) * static_cast<size_t>(n);
    const void* src = d.dist.p;
    if (d.dev != d0.dev) {  // the block crosses to the first device
      if (peer.bytes < slots * w) SF_TRY(peer.alloc(d0.dev, slots * w, "peer stripes"));
      SF_CUDA(cudaMemcpyPeerAsync(peer.p, d0.dev, d.dist.p, d.dev, slots * w, st));
      src = peer.p;
    }
    const int blocks = grid_for(static_cast<int64_t>(slots), 256);
    if (plan->prec == SF_FP64)
      condense_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(src), n, d.a, d.b,
                                                      mat.as<double>(), bad.as<int>());
    else
      condense_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(src), n, d.a, d.b,
                                                     mat.as<double>(), bad.as<int>());
    SF_CUDA(cudaGetLastError());
    if (d.dev != d0.dev) SF_CUDA(cudaStreamSynchronize(st));  // the peer buffer is reused
  }
  diagonal_zero_kernel<<<grid_for(n, 256), 256, 0, st>>>(mat.as<double>(), n);
  SF_CUDA(cudaGetLastError());
  int flag = 0;
  SF_CUDA(cudaMemcpyAsync(&flag, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  if (flag) return fail(SF_EINVAL, "condense: duplicated slot disagrees");
  if (host_pinned(out)) {
    SF_CUDA(cudaMemcpyAsync(out, mat.p, nn * 8, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
  } else {
    SF_TRY(staged_d2h(d0.dev, st, mat.as<char>(), reinterpret_cast<char*>(out), nn * 8, copy_threads(1)));
  }
  return SF_OK;
}

// compute_distance_matrix (kernels.hpp:319-326): full-range plan, finalize,
// condense on device, one copy of the n x n matrix to the caller.
sf_status sf_compute_distance_matrix(const sf_problem* p, sf_metric metric, sf_precision prec, double* out,
                                     const sf_exec* ex, sf_stats* stats_out) {
  if (!out) return fail(SF_EINVAL, "out is null");
  if (!p) return fail(SF_EINVAL, "problem is null");
  sf_plan* plan = nullptr;
  SF_TRY(sf_plan_create(p, metric, prec, 0, -1, ex, &plan));
  std::unique_ptr<sf_plan> guard(plan);
  SF_TRY(sf_plan_run(plan, 1));
  SF_TRY(sf_plan_condense(plan, out));
  if (stats_out) *stats_out = plan->stats;
  return SF_OK;
}

// ---------------------------------------------------------------- Mantel
namespace {
std::uint64_t mantel_mix64(std::uint64_t x) {  // splitmix64, validate.cpp:101-106
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// The reference's permutation p (validate.cpp:133-136): same engine, same
// std::shuffle (this host code is built with the same C++ library).
void mantel_perm(int32_t n, std::uint64_t seed, int32_t p, int32_t* out) {
  std::vector<int> perm(static_cast<std::size_t>(n));
  std::mt19937_64 rng(mantel_mix64(seed ^ mantel_mix64(static_cast<std::uint64_t>(p) + 1)));
  std::iota(perm.begin(), perm.end(), 0);
  std::shuffle(perm.begin(), perm.end(), rng);
  std::copy(perm.begin(), perm.end(), out);
}
}  // namespace

sf_status sf_mantel_permutation(int32_t n, uint64_t seed, int32_t p, int32_t* perm_out) {
  if (n < 1 || p < 0 || !perm_out) return fail(SF_EINVAL, "mantel_permutation: bad argument");
  mantel_perm(n, seed, p, perm_out);
  return SF_OK;
}

sf_status sf_mantel(int32_t n, const double* m1, const double* m2, int32_t permutations, uint64_t seed,
                    int32_t device, double* r_out, double* p_value_out) {
  if (permutations < 1) return fail(SF_EINVAL, "mantel: need at least 1 permutation");
  if (!m1 || !m2 || !r_out || !p_value_out) return fail(SF_EINVAL, "null argument");
  if (n < 2) return fail(SF_EINVAL, "distance matrix needs at least 2 samples");
  sf_exec ex{};
  ex.n_devices = 1;
  ex.devices = &device;
  std::vector<int> devs;
  SF_TRY(usable_devices(&ex, devs));
  SF_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  SF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{st};
  const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);
  const int32_t nrp = (n + 1) / 2;  // row pairs {i, n-1-i}
  DevBuf dx, dy, dpart, dpxy, dasym, ddot, dperm, dpp;
  SF_TRY(dx.alloc(device, nn * 8, "mantel matrix 1"));
  SF_TRY(dy.alloc(device, nn * 8, "mantel matrix 2"));
  SF_TRY(dpart.alloc(device, static_cast<size_t>(nrp) * 16, "mantel partials"));
  SF_TRY(dpxy.alloc(device, static_cast<size_t>(nrp) * 8, "mantel cross partials"));
  SF_TRY(dasym.alloc(device, 16, "asymmetry flag"));
  SF_TRY(ddot.alloc(device, static_cast<size_t>(permutations + 1) * 8, "permutation cross terms"));
  SF_CUDA(cudaMemcpyAsync(dx.p, m1, nn * 8, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(dy.p, m2, nn * 8, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemsetAsync(dasym.p, 0xff, 16, st));
  std::vector<double> part(static_cast<size_t>(nrp) * 2);
  // pass 1: means (+ symmetry, as condensed_upper checks, validate.cpp:87-91)
  mt_stats_kernel<<<nrp, kMantelThreads, 0, st>>>(dx.as<double>(), dy.as<double>(), n, 0, 0.0, 0.0,
                                                  dpart.as<double>(), dpxy.as<double>(),
                                                  dasym.as<unsigned long long>());
  SF_CUDA(cudaGetLastError());
  unsigned long long asym[2];
  SF_CUDA(cudaMemcpyAsync(asym, dasym.p, 16, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaMemcpyAsync(part.data(), dpart.p, part.size() * 8, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  for (int m = 0; m < 2; ++m)
    if (asym[m] != ~0ull)
      return fail(SF_EINVAL, "distance matrix is asymmetric at (" + std::to_string(asym[m] / static_cast<unsigned>(n)) +
                                 "," + std::to_string(asym[m] % static_cast<unsigned>(n)) + ")");
  const double cnt = static_cast<double>(n) * static_cast<double>(n - 1) / 2.0;
  double sx = 0.0, sy = 0.0;
  for (int32_t i = 0; i < nrp; ++i) {
    sx += part[2 * static_cast<size_t>(i)];
    sy += part[2 * static_cast<size_t>(i) + 1];
  }
  const double mx = sx / cnt, my = sy / cnt;
  // pass 2: sxx, syy (host-ordered) and the sxy partials (device-reduced like
  // every permutation's cross term)
  mt_stats_kernel<<<nrp, kMantelThreads, 0, st>>>(dx.as<double>(), dy.as<double>(), n, 1, mx, my,
                                                  dpart.as<double>(), dpxy.as<double>(),
                                                  dasym.as<unsigned long long>());
  mt_reduce_kernel<<<1, kMantelThreads, 0, st>>>(dpxy.as<double>(), nrp, ddot.as<double>() + permutations);
  SF_CUDA(cudaGetLastError());
  SF_CUDA(cudaMemcpyAsync(part.data(), dpart.p, part.size() * 8, cudaMemcpyDeviceToHost, st));
  double sxy = 0.0;
  SF_CUDA(cudaMemcpyAsync(&sxy, ddot.as<double>() + permutations, 8, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  double sxx = 0.0, syy = 0.0;
  for (int32_t i = 0; i < nrp; ++i) {
    sxx += part[2 * static_cast<size_t>(i)];
    syy += part[2 * static_cast<size_t>(i) + 1];
  }
  if (sxx <= 0.0 || syy <= 0.0)
    return fail(SF_EINVAL, "mantel: a distance matrix has zero variance, correlation is undefined");
  const double denom = std::sqrt(sxx * syy);
  const double r = sxy / denom;

  // permutations in batches; the next batch is generated on host threads
  // while the device works on the current one
  const int32_t B = static_cast<int32_t>(std::max<int64_t>(
      1, std::min<int64_t>({permutations, 65535, (int64_t{256} << 20) / (4 * static_cast<int64_t>(n))})));
  SF_TRY(dperm.alloc(device, static_cast<size_t>(B) * n * 4, "permutations"));
  SF_TRY(dpp.alloc(device, static_cast<size_t>(B) * nrp * 8, "permutation partials"));
  int32_t* hperm = nullptr;
  SF_CUDA(cudaMallocHost(&hperm, static_cast<size_t>(2) * B * n * 4));
  struct HostGuard {
    int32_t* p;
    ~HostGuard() { cudaFreeHost(p); }
  } hguard{hperm};
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto generate = [&](int32_t p0, int32_t cnt_p, int32_t* dst) {
    std::vector<std::thread> pool;
    const int32_t T = static_cast<int32_t>(std::min<unsigned>(hw, static_cast<unsigned>(cnt_p)));
    for (int32_t t = 0; t < T; ++t)
      pool.emplace_back([=] {
        for (int32_t q = t; q < cnt_p; q += T) mantel_perm(n, seed, p0 + q, dst + static_cast<int64_t>(q) * n);
      });
    for (auto& th : pool) th.join();
  };
  generate(0, std::min(B, permutations), hperm);
  for (int32_t p0 = 0, buf = 0; p0 < permutations; p0 += B, buf ^= 1) {
    const int32_t cnt_p = std::min(B, permutations - p0);
    int32_t* cur = hperm + static_cast<int64_t>(buf) * B * n;
    SF_CUDA(cudaMemcpyAsync(dperm.p, cur, static_cast<size_t>(cnt_p) * n * 4, cudaMemcpyHostToDevice, st));
    mt_perm_kernel<<<dim3(static_cast<unsigned>(cnt_p), static_cast<unsigned>(nrp)), kMantelThreads, 0, st>>>(
        dx.as<double>(), dy.as<double>(), n, mx, my, dperm.as<int32_t>(), nrp, dpp.as<double>());
    mt_reduce_kernel<<<cnt_p, kMantelThreads, 0, st>>>(dpp.as<double>(), nrp, ddot.as<double>() + p0);
    SF_CUDA(cudaGetLastError());
    if (p0 + B < permutations)  // overlaps the kernels just queued
      generate(p0 + B, std::min(B, permutations - p0 - B), hperm + static_cast<int64_t>(buf ^ 1) * B * n);
    SF_CUDA(cudaStreamSynchronize(st));  // the other buffer is reused next
  }
  std::vector<double> dot(static_cast<size_t>(permutations));
  SF_CUDA(cudaMemcpy(dot.data(), ddot.p, dot.size() * 8, cudaMemcpyDeviceToHost));
  int exceed = 0;
  for (double v : dot)
    if (v / denom >= r) ++exceed;
  *r_out = r;
  *p_value_out = (1.0 + exceed) / (1.0 + permutations);
  return SF_OK;
}

// ---------------------------------------------------------------- .strf
// write_stripe_file (stripes.cpp:179-201) straight from the plan's device
// stripes: 32-byte header, finalized distances then raw totals (UW, WN),
// FNV-1a 64 (common.cpp:51-58) over the payload. Blocks stream through two
// pinned staging buffers: the next block's D2H copy overlaps hashing and
// writing the current one.
sf_status sf_plan_write_strf(sf_plan* plan, const char* path) {
  if (!plan || !path) return fail(SF_EINVAL, "null argument");
  if (!plan->ran) return fail(SF_ESTATE, "plan has not run");
  if (!plan->finalized) return fail(SF_EINVAL, "refusing to write an unfinalized stripe set");
  if (plan->metric == SF_GENERALIZED)
    return fail(SF_EINVAL, "generalized stripes have no .strf metric code");
  SF_TRY(sf_plan_sync(plan));
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(SF_EINVAL, std::string("cannot open '") + path + "' for writing");
  struct FileGuard {
    FILE* f;
    ~FileGuard() {
      if (f) std::fclose(f);
    }
  } fguard{f};
  const size_t w = plan->prec == SF_FP64 ? 8 : 4;
  unsigned char hdr[32] = {'S', 'T', 'R', 'F', 1, static_cast<unsigned char>(w),
                           static_cast<unsigned char>(plan->metric), 0};
  const uint64_t dims[3] = {static_cast<uint64_t>(plan->n), static_cast<uint64_t>(plan->start),
                            static_cast<uint64_t>(plan->stop)};
  for (int i = 0; i < 3; ++i)
    for (int b = 0; b < 8; ++b) hdr[8 + 8 * i + b] = static_cast<unsigned char>(dims[i] >> (8 * b));
  bool ok = std::fwrite(hdr, 1, 32, f) == 32;
  // blocks: every device's distances, then (ratio metrics) every device's totals
  struct Block {
    DeviceState* d;
    const char* src;
    size_t bytes;
  };
  std::vector<Block> blocks;
  const bool has_t = plan->metric != SF_WEIGHTED_UNNORMALIZED;
  for (int arr = 0; arr < (has_t ? 2 : 1); ++arr)
    for (auto& dp : plan->devs) {
      const size_t bytes = static_cast<size_t>(dp->b - dp->a) * plan->n * w;
      blocks.push_back({dp.get(), arr == 0 ? dp->dist.as<char>() : dp->tot.as<char>(), bytes});
    }
  constexpr size_t CH = size_t{64} << 20;
  char* stage = nullptr;
  SF_CUDA(cudaMallocHost(&stage, 2 * CH));
  struct HostGuard {
    char* p;
    ~HostGuard() { cudaFreeHost(p); }
  } hguard{stage};
  // one event pair per device: an event must be recorded on a stream of the
  // device it was created on (chunks of several devices alternate buffers)
  struct DevEvents {
    int dev = -1;
    cudaEvent_t ev[2] = {nullptr, nullptr};
  };
  std::vector<DevEvents> evs(plan->devs.size());
  struct EventGuard {
    std::vector<DevEvents>& e;
    ~EventGuard() {
      for (auto& x : e)
        for (auto ev : x.ev)
          if (ev) {
            cudaSetDevice(x.dev);
            cudaEventDestroy(ev);
          }
    }
  } eguard{evs};
  for (size_t i = 0; i < plan->devs.size(); ++i) {
    evs[i].dev = plan->devs[i]->dev;
    SF_CUDA(cudaSetDevice(evs[i].dev));
    for (auto& ev : evs[i].ev) SF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  auto dev_index = [&](const DeviceState* d) {
    for (size_t i = 0; i < plan->devs.size(); ++i)
      if (plan->devs[i].get() == d) return i;
    return size_t{0};
  };
  // flatten into chunks, issue chunk i+1 before consuming chunk i
  struct Chunk {
    DeviceState* d;
    const char* src;
    size_t len;
  };
  std::vector<Chunk> chunks;
  for (const Block& b : blocks)
    for (size_t off = 0; off < b.bytes; off += CH) chunks.push_back({b.d, b.src + off, std::min(CH, b.bytes - off)});
  auto event_of = [&](size_t i) { return evs[dev_index(chunks[i].d)].ev[i & 1]; };
  auto issue = [&](size_t i) -> sf_status {
    const Chunk& c = chunks[i];
    SF_CUDA(cudaSetDevice(c.d->dev));
    SF_CUDA(cudaMemcpyAsync(stage + (i & 1) * CH, c.src, c.len, cudaMemcpyDeviceToHost, c.d->stream));
    SF_CUDA(cudaEventRecord(event_of(i), c.d->stream));
    return SF_OK;
  };
  uint64_t h = 0xcbf29ce484222325ull;
  if (!chunks.empty()) SF_TRY(issue(0));
  for (size_t i = 0; i < chunks.size(); ++i) {
    SF_CUDA(cudaEventSynchronize(event_of(i)));
    if (i + 1 < chunks.size()) SF_TRY(issue(i + 1));  // other buffer: free since chunk i-1 was consumed
    const unsigned char* p = reinterpret_cast<const unsigned char*>(stage + (i & 1) * CH);
    for (size_t k = 0; k < chunks[i].len; ++k) {
      h ^= p[k];
      h *= 0x100000001b3ull;
    }
    ok = ok && std::fwrite(p, 1, chunks[i].len, f) == chunks[i].len;
  }
  unsigned char tail[8];
  for (int b = 0; b < 8; ++b) tail[b] = static_cast<unsigned char>(h >> (8 * b));
  ok = ok && std::fwrite(tail, 1, 8, f) == 8;
  ok = (std::fclose(f) == 0) && ok;
  fguard.f = nullptr;
  if (!ok) return fail(SF_EINVAL, std::string("failed writing '") + path + "'");
  return SF_OK;
}

}  // extern "C"
