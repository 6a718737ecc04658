/*
 * zsort_b200.h -- C ABI of the B200-native stable z-score partitioning sort.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (arxiv 2605.14419, Python package `zsort`) has no C ABI of its own: its
 * native boundary is the numba dispatcher call
 *     _kernels.zsort_driver(src_k, src_c, out_k, out_c, scr_k, scr_c, k,
 *                           scale, mean, std, zmin, insertion_limit,
 *                           counting_limit, depth_guard, counters)
 * (/root/reference/pkg/src/zsort/_kernels.py:393-396) reached from
 * core.zsort (core.py:348-400).  The entry points below replace that
 * boundary with plain pointers and sizes; every pointer named d_* is CUDA
 * device memory owned by the caller, and every call is stream-ordered on the
 * given cudaStream_t (passed as void* so this header needs no CUDA include).
 *
 * Conventions (mirroring the reference):
 *  - inputs are never modified (core.py:351-352);
 *  - outputs and workspace are caller-allocated; kernels never allocate
 *    (_kernels.py:3-5);
 *  - reentrant: a call's state lives in its workspace;
 *    the library keeps only per-host-thread state (a pinned control-block
 *    mirror, two events and a side stream per thread, created at first use)
 *    and once-per-device kernel attributes (shared-memory opt-in, the team
 *    kernel's resident-cluster count) guarded by mutexes, so concurrent
 *    calls from different host threads on their own streams and workspaces
 *    are independent (tests/test_gpu_contract.py::TestConcurrency); nothing
 *    reads the environment (tuning constants are compile-time);
 *  - return 0 on success or a ZSB_ERR_* code; zsb_last_error() gives a
 *    thread-local message.  The Python wrapper maps ZSB_ERR_ARG/ZSB_ERR_NAN
 *    to ValueError and ZSB_ERR_DTYPE to TypeError, like core.py:151-181.
 */
#ifndef ZSORT_B200_H
#define ZSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Key element types.  The reference accepts only signed integers
 * (core.py:151-165); float64 is a documented extension (NaN rejected). */
typedef enum { ZSB_KEY_I64 = 0, ZSB_KEY_F64 = 1 } zsb_key_dtype;

/* Bucket mapping for partition levels.
 *  ZSB_MAP_FITTED: z-score mapping whose scale is fitted to the segment's
 *                  z-range (GPU default: balanced buckets, fewer levels);
 *  ZSB_MAP_PAPER:  the paper's Eq. 1 exactly, scale = k/4 with
 *                  k = max(2, round(alpha*sqrt(n))) (core.py:146-148,233-234).
 * Both produce the identical (unique) stable order. */
typedef enum { ZSB_MAP_FITTED = 0, ZSB_MAP_PAPER = 1 } zsb_mapping;

/* Mirror of SortConfig (core.py:63-89) plus the GPU mapping choice. */
typedef struct {
    double alpha;                     /* (0, 2]; paper-mode bucket count */
    int64_t insertion_threshold;      /* n <= this: one shared-memory finish */
    int64_t counting_range_threshold; /* accepted for API parity */
    int64_t depth_guard;              /* >= 3: levels before the exact bit split */
    int32_t collect_stats;            /* accepted; counters are always kept */
    int32_t mapping;                  /* zsb_mapping */
} zsb_config;

/* SortStats slots (core.py:135-143, _kernels.py:16-21). */
enum {
    ZSB_STAT_MAX_DEPTH = 0,
    ZSB_STAT_FALLBACKS = 1,
    ZSB_STAT_COUNTING = 2,
    ZSB_STAT_INSERTION = 3,
    ZSB_STAT_SCATTERS = 4,
    ZSB_STAT_SLOTS = 5
};

enum {
    ZSB_OK = 0,
    ZSB_ERR_ARG = 1,       /* bad size/pointer/config (ValueError) */
    ZSB_ERR_DTYPE = 2,     /* unsupported key or payload type (TypeError) */
    ZSB_ERR_NAN = 3,       /* NaN key (ValueError) */
    ZSB_ERR_WORKSPACE = 4, /* workspace too small */
    ZSB_ERR_CUDA = 5       /* CUDA launch/runtime failure (RuntimeError) */
};

/* Bytes of device workspace zsb_sort needs for n keys.
 * Replaces the scratch arrays allocated at core.py:367-368,393-394. */
size_t zsb_workspace_bytes(int64_t n, int32_t key_dtype, int32_t payload_bytes, const zsb_config *cfg);

/* Stable ascending sort of n 8-byte keys with an optional 4- or 8-byte
 * payload (payload_bytes 0/4/8; d_payload/d_out_payload may be NULL when 0).
 * Replaces core.zsort -> _kernels.zsort_driver (core.py:348-400,
 * _kernels.py:393-450).  h_stats (may be NULL) receives ZSB_STAT_SLOTS
 * int64 counters; with h_stats the call blocks until the sort has completed.
 * With h_stats == NULL the call is stream-ordered: it returns once the last
 * partition level is enqueued on `stream` (a sort with several levels still
 * waits on the host for each level's outcome), so callers synchronise on
 * the stream like after any CUDA library call. */
int zsb_sort(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, void *d_out_keys,
             void *d_out_payload, int64_t n, const zsb_config *cfg, void *d_workspace, size_t workspace_bytes,
             int64_t *h_stats, void *stream);

/* zsort_rec (core.py:403-437 -> _kernels.zsort_rec_driver, _kernels.py:453-473):
 * stable sort of one segment in the recursion phase, given the caller's
 * bucket count k (clamped to one pass's fan-out, 2048), scale and estimated
 * mean.  The segment starts at level depth + 1: one fused pass gathers min,
 * max and the squared deviation around mean_est (_kernels.py:74-88), then
 * Eq. 1 with (mean_est, std, zmin = |min - mean_est| / std, scale) buckets it;
 * deeper levels size k to their segments like zsb_sort.  Validation as
 * core.py:416-424: depth >= 1, k >= 2, scale > 0, n > insertion_threshold
 * (ZSB_ERR_ARG).  Workspace: zsb_rec_workspace_bytes. */
size_t zsb_rec_workspace_bytes(int64_t n, int32_t key_dtype, int32_t payload_bytes, int64_t k);
int zsb_sort_rec(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes,
                 void *d_out_keys, void *d_out_payload, int64_t n, int64_t k, double scale, double mean_est,
                 int64_t depth, const zsb_config *cfg, void *d_workspace, size_t workspace_bytes, int64_t *h_stats,
                 void *stream);

/* Grid-wide moments of n keys (north-star subsystem 1; replaces
 * first_pass + variance_pass, _kernels.py:28-71, core.py:184-234).
 * h_out[0..7] = count, mean, M2 (sum of squared deviations around the mean),
 * min, max (as doubles), 0, 0, NaN count.  h_limbs[0..1] = the exact int64
 * key sum as first_pass limbs (value = hi*2^32 + lo; int64 keys only), and
 * h_min_max_bits[0..1] = the raw 8-byte min and max keys.  The mean of int64
 * keys is the correctly rounded quotient of the exact sum (core.py:226).
 * Uses the front of a zsb_workspace_bytes(n, ...) workspace; blocks. */
int zsb_moments(const void *d_keys, int32_t key_dtype, int64_t n, void *d_workspace, size_t workspace_bytes,
                double *h_out, int64_t *h_limbs, uint64_t *h_min_max_bits, void *stream);

/* Parameter-injected bucket histogram (north-star subsystem 2; replaces
 * histogram_pass/build_partition_plan, _kernels.py:91-112, core.py:248-256):
 * params = {mean, std, zmin, scale}; d_counts receives k int64 counts. */
int zsb_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k,
                  int64_t *d_counts, void *d_workspace, size_t workspace_bytes, void *stream);

/* Parameter-injected one-level stable scatter into bucket order
 * (north-star subsystems 3+4; replaces exclusive_offsets + scatter_pass,
 * _kernels.py:115-133, core.py:259-276). */
int zsb_scatter(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, int64_t n,
                const double *params, int64_t k, void *d_out_keys, void *d_out_payload, void *d_workspace,
                size_t workspace_bytes, void *stream);

/* Structural stable-permutation check on the device (K8; replaces
 * verify.check_stable_permutation, verify.py:55-108, for the case
 * payload = original index): returns through h_result the number of
 * violations of (sorted, permutation, key match, stability); 0 = stable.
 * d_index is int64 (index_bytes 8) or int32 (4); d_in_keys is the unsorted
 * input.  Needs zsb_check_workspace_bytes(n) of workspace. */
size_t zsb_check_workspace_bytes(int64_t n);
int zsb_check_sorted(const void *d_in_keys, const void *d_out_keys, const void *d_index, int32_t index_bytes,
                     int32_t key_dtype, int64_t n, int64_t index_base, void *d_workspace, int64_t *h_result,
                     void *stream);

/* ---- multi-GPU phases (one process per GPU; the NCCL collectives D1-D3 run
 * between these calls from paper_2605_14419_b200/dist.py over
 * torch.distributed).  All are stream-ordered on `stream`. ---- */

/* D1 payload, one pass over the shard: d_out4 = {count, sum(x - c),
 * sum((x - c)^2), c} (double) with c = shift, or the shard's first key when
 * shift is NaN, and d_out_bits2 = ordered (order-preserving uint64) min and
 * max of the local shard; both are initialised by the call.  The ranks
 * combine the four values with Chan's merge.  Replaces first_pass +
 * variance_pass (_kernels.py:28-71) for a shard. */
int zsb_local_moments(const void *d_keys, int32_t key_dtype, int64_t n, double shift, double *d_out4,
                      uint64_t *d_out_bits2, void *stream);

/* Index of the `occurrence`-th (0-based) local record whose key equals the
 * key with bits key_bits (-0.0 and +0.0 are one key), or -1: the record a
 * cut inside a one-valued run falls on.  Workspace of
 * zsb_occurrence_workspace_bytes(); blocks until done. */
size_t zsb_occurrence_workspace_bytes(void);

/* Counter-based generator of the reference's key families on the device
 * (datagen.py:92-162 shapes; gen_kernels.cuh): family 0 uniform, 1 normal,
 * 2 skewed (Pareto), 3 nearly_sorted, 4 high_duplicate.  Writes the int64
 * keys of global positions [offset, offset + n) of an n_total-key workload
 * to d_out; key i depends only on (family, seed, i, params), so shards and
 * checkers regenerate any key independently.  params (may be NULL for the
 * reference defaults) = {normal_mu, normal_sigma, pareto_alpha, pareto_xm,
 * swap_fraction, dup_range}.  Stream-ordered. */
int zsb_generate(int32_t family, int64_t offset, int64_t n, int64_t n_total, uint64_t seed, const double *params,
                 int64_t *d_out, void *stream);
int zsb_occurrence_index(const void *d_keys, int32_t key_dtype, int64_t n, uint64_t key_bits, int64_t occurrence,
                         void *d_workspace, int64_t *h_index, void *stream);

/* D2 payload: histogram of the k global z-score buckets (params = {center,
 * std, zmin, scale}, Eq. 1, _kernels.py:91-112) into d_counts (int64[k],
 * zeroed by the call), k <= 16384. */
int zsb_bucket_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k,
                         int64_t *d_counts, void *stream);

/* Ordered min/max of the local keys falling in each of nb (<= 32)
 * candidate buckets (all-equal test before a cut inside a bucket). */
int zsb_bucket_minmax(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k, int32_t nb,
                      const int32_t *d_buckets, uint64_t *d_omin, uint64_t *d_omax, void *stream);

/* Refinement histograms for a cut that falls inside a bucket: for each of
 * nq (<= 32) queries, counts the local records with bucket == d_qbucket[q]
 * and ordered key in [d_qlo[q], d_qhi[q]] by the exact digit
 * (ord - d_qlo[q]) >> d_qshift[q] into d_counts[q*nbins + digit] (int64,
 * zeroed by the call). */
int zsb_range_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k, int32_t nq,
                        const int32_t *d_qbucket, const uint64_t *d_qlo, const uint64_t *d_qhi, const int32_t *d_qshift,
                        int32_t nbins, int64_t *d_counts, void *stream);

/* D3 input: stable partition of the local shard into ncuts+1 destination
 * ranks.  Record i (global index gidx_base + i) goes to the number of cuts
 * c_j with (bucket(x), ord(x), gidx) >= (h_cut_bucket[j], h_cut_ord[j],
 * h_cut_gidx[j]) lexicographically -- the global stable order -- so every
 * destination receives its records in input order.  h_part_counts receives
 * the ncuts+1 per-destination counts; blocks until done. */
size_t zsb_partition_workspace_bytes(int64_t n, int32_t payload_bytes, int32_t nparts);
int zsb_partition_to_ranks(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes,
                           int64_t n, const double *params, int64_t k, int64_t gidx_base, int32_t ncuts,
                           const int32_t *h_cut_bucket, const uint64_t *h_cut_ord, const int64_t *h_cut_gidx,
                           void *d_out_keys, void *d_out_payload, int64_t *h_part_counts, void *d_workspace,
                           size_t workspace_bytes, void *stream);

/* Fused exchange (paper_2605_14419_b200/dist.py, exchange="p2p").  First
 * zsb_partition_to_ranks with d_out_keys = NULL: the destination counts
 * only (histogram + scan left in the workspace).  Then zsb_partition_send on
 * the same workspace: the stable partition's scatter writes the records of
 * destination d straight into d's receive buffers h_dest_keys[d] /
 * h_dest_payload[d] (device addresses; other ranks' buffers are CUDA IPC
 * mappings, so the stores cross NVLink) starting at h_dest_offset[d] = the
 * records of d from lower-ranked sources -- the exchange happens inside the
 * partition kernel, with no send buffer and no all_to_all.  Blocks until the
 * stores are done; the caller synchronises the ranks before reading. */
int zsb_partition_send(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, int64_t n,
                       int32_t nparts, const uint64_t *h_dest_keys, const uint64_t *h_dest_payload,
                       const int64_t *h_dest_offset, void *d_workspace, size_t workspace_bytes, void *stream);

/* Optional per-phase device timing of zsb_sort on the calling thread (CUDA
 * events around each launch group, on the sort's own stream).  Phase slots:
 * 0 moments, 1 histogram, 2 scan, 3 scatter, 4 classify+plan, 5 finish,
 * 6 recursion moments+params, 7 misc.  zsb_timing_read fills up to nslots
 * accumulated milliseconds and kernel-launch counts (launch counts are kept
 * even when timing is off) and returns the number of slots. */
void zsb_timing_enable(int32_t on);
int32_t zsb_timing_read(double *ms, int64_t *launches, int32_t nslots, int32_t reset);
/* Records each phase's launches have passed over since the last reset (slots
 * 1 histogram and 3 scatter: the level's records, every level; 5 finish: n
 * per sort); bench.py's per-launch roofline uses them.  Read before the
 * zsb_timing_read call that resets. */
int32_t zsb_timing_records(int64_t *records, int32_t nslots);

/* Thread-local message for the last failing call. */
const char *zsb_last_error(void);

/* Bounds-check builds (-DZSB_CHECKS, tools/bounds_check.py): the number of
 * out-of-range shared/global indices the data-path kernels have seen on this
 * device since the last reset (synchronises the device); -1 in normal
 * builds. */
int64_t zsb_check_violations(int32_t reset);

/* Build/version string (compile flags and target arch). */
const char *zsb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ZSORT_B200_H */
