/*
 * ddks.h — C ABI of the B200-native exact ddKS library (libddks.so).
 *
 * The statistic (PAPER.md = the arxiv 2106.13706 text; P:L<n> = its line n):
 *   P:L33-35 (§2.1, Eq. 1)   D = max |C_P(x) - C_T(x)|, C = orthant occupancy about x.
 *   P:L40-44 (§2.1, Eq. 2)   evaluated at every point of both samples (pooled origins: P rows, then Q rows).
 *   P:L59-67 (§2.2.1, Eq. 3) orthant bit k = [x_k >= o_k] (element-wise "greater than or equal"; ties
 *                            and the origin itself fall on the >= side; reading R1).
 *   P:L78-81 (Eq. 6), P:L238 per-sample normalised difference |c_P/n_P - c_Q/n_Q| (reading R2), kept exact as
 *                            num = max_o max_q |c_P[q]*n_Q - c_Q[q]*n_P|,  den = n_P*n_Q,  D = (double)num/(double)den.
 *   P:L371 (§4.2)            permutation test; p = (1 + #{null_num >= observed_num}) / (1 + n_perm) (reading R9).
 *
 * Conventions shared by every call:
 *   - Points are float32, row-major, contiguous: a sample of n points in d dimensions is n*d floats.
 *   - Input pointers may be DEVICE pointers (read in place) or HOST pointers (copied to the device on
 *     `stream` inside the call; this is what the end-to-end measurement times). The kind is detected with
 *     cudaPointerGetAttributes. Inputs are caller-owned and only read; they must stay valid until the call returns.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). It is borrowed, never destroyed.
 *   - Every call is synchronous with respect to its host outputs (it synchronises `stream` before returning).
 *   - Results go to caller-owned HOST memory.
 *   - Nothing throws or aborts across the ABI; every call returns a ddks_status. On error the host outputs are
 *     unspecified and ddks_last_error(ctx) holds a one-line message.
 *   - A context is bound to one device and one host thread; it is not thread-safe.
 *   - Multi-GPU (world > 1): every rank makes the same call with the same (replicated) inputs.
 *       ddks_stat /              shard the pooled ORIGINS -- `world` contiguous ranges of the pooled order, or, when
 *       ddks_significance        the kd-ordered count runs (2 <= d <= 8 and N large enough), the origin blocks r,
 *                                r + world, r + 2 world, ... of the kd order (every rank computes the same order).
 *                                ddks_stat combines with ONE collective: an ncclAllGather of every rank's 32-byte record
 *                                {num, argmax candidate, flags}, reduced on the host by ddks_combine_records; the
 *                                significance all-reduces num, the argmax candidate, the flags and its M_T histogram.
 *       ddks_stat_batch /
 *       ddks_permutation_null    shard ITEMS (pairs / permutations) contiguously and gather the per-item nums plus the
 *                                rank's flags in ONE ncclAllGather of records padded to the largest shard (unpadded on
 *                                the host by ddks_unpad_items), so every rank returns the full result.
 *       ddks_vdks / ddks_rdks    shard points + voxels / corners (see each call).
 *   - Limits: 1 <= d <= 8 (ddks_rdks: any d >= 1); n_P, n_Q >= 1; n_P + n_Q < 2^31; n_P*n_Q < 2^53 (so D is one
 *     exact IEEE division).
 *   - Results do not depend on the world size, the stream, the flags marked TEST ONLY, or which internal kernel ran.
 */
#ifndef DDKS_H_
#define DDKS_H_

#include <stdint.h>

#if defined(__GNUC__)
#define DDKS_API __attribute__((visibility("default")))
#else
#define DDKS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ddks_ctx ddks_ctx; /* opaque: owns device workspace and (world > 1) an NCCL communicator */

typedef enum {
    DDKS_OK = 0,
    DDKS_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative size, B < 1, n_perm < 0, bad flags, bad rank/world */
    DDKS_ERR_EMPTY_SAMPLE = 2,     /* n_P == 0 || n_Q == 0            (SPEC core-types EmptySample)        */
    DDKS_ERR_DIM_UNSUPPORTED = 3,  /* d < 1 || d > 8                                                         */
    DDKS_ERR_NONFINITE = 4,        /* a NaN or +-Inf coordinate        (SPEC core-types NonFiniteValue)     */
    DDKS_ERR_TOO_LARGE = 5,        /* n_P + n_Q >= 2^31 or n_P*n_Q >= 2^53                                  */
    DDKS_ERR_CUDA = 6,             /* a CUDA runtime error (message in ddks_last_error)                     */
    DDKS_ERR_NCCL = 7,             /* an NCCL error                                                          */
    DDKS_ERR_OOM = 8               /* device workspace allocation failed                                    */
} ddks_status;

/* Flags for ddks_create. */
#define DDKS_FLAG_DEFAULT 0u
#define DDKS_FLAG_NO_VALIDATE 1u /* skip the NaN/Inf check (inputs are still packed and -0 canonicalised)  */
#define DDKS_FLAG_TIES_GT 2u     /* TEST ONLY: bit k = [x_k > o_k] instead of >= (shows the convention matters) */
#define DDKS_FLAG_FORCE_DIRECT 4u /* TEST ONLY: never split the point axis into segments (exercises the in-kernel
                                     finalisation at small N; results are identical either way)              */
#define DDKS_FLAG_PERM_GATHER 16u /* TEST ONLY: permutation null by gathering each relabelled sample and re-running the
                                      full classification (the default label-invariant path classifies each pair once
                                      for a chunk of permutations; both give identical results)                    */
#define DDKS_FLAG_NO_X0 32u        /* TEST ONLY: never use the kd-ordered count (ddks_stat / ddks_significance reorder the
                                      pooled points hierarchically by x_0 .. x_{K-1} when 2 <= d <= 8 and N >= 80000, 
                                      so whole tiles share those bits; identical results)                          */
#define DDKS_FLAG_FORCE_X0 64u     /* TEST ONLY: use the kd-ordered count for any N (2 <= d <= 8)                      */
#define DDKS_FLAG_KD_SHIFT 16u     /* TEST ONLY: bits 16..18 = K in 1..4 force the number of kd levels (0: cost model;
                                      K is capped at d and at the deepest level built, 4)                           */
#define DDKS_FLAG_KD_LEVELS(k) (((unsigned)(k) & 7u) << DDKS_FLAG_KD_SHIFT)
#define DDKS_FLAG_NO_GRAPH 4096u   /* never capture a call into a CUDA graph (by default the second identical call of
                                      ddks_stat, ddks_stat_batch, ddks_permutation_null, ddks_vdks or ddks_rdks -- same
                                      input pointers, sizes, flags and workspace -- is captured and later calls replay
                                      it with one cudaGraphLaunch; identical results; host inputs must then be pinned) */
#define DDKS_FLAG_NCCL_SELF 2048u  /* TEST ONLY (world == 1): create a one-rank NCCL communicator and run every collective
                                      of the multi-GPU path (all-reduce / all-gather) through it; identical results */
#define DDKS_FLAG_RDKS_FULL_SORT 128u /* TEST ONLY: ddks_rdks sorts every key (8-pass radix sort) instead of the bucket-pruned
                                         sweep that sorts only the buckets able to hold the maximum; identical results */
#define DDKS_FLAG_NO_RANK 256u    /* TEST ONLY: never use the rank-lane count (ddks_stat at d = 3 and d = 5..8 and mid N
                                      compares each pair's coordinates as 10-bit per-CTA rank lanes, ceil(d/3) integer
                                      adds per pair, instead of d FP32 compares; identical results)                 */
#define DDKS_FLAG_FORCE_RANK 512u /* TEST ONLY: the rank-lane count at every 2 <= d <= 8 and every N > 8192 (DIFF counters
                                      when max(n_P, n_Q) / gcd <= 7, else SPLIT in two launches; also for
                                      ddks_significance); identical results                                          */
#define DDKS_FLAG_PROFILE 8u      /* record CUDA events around every count-kernel launch (see ddks_profile_read) */

typedef struct {
    uint64_t num;          /* max over origins and orthants of |c_P*n_Q - c_Q*n_P| (exact integer)            */
    uint64_t den;          /* n_P * n_Q                                                                         */
    double D;              /* (double)num / (double)den, one IEEE-754 round-to-nearest-even division           */
    int64_t argmax_origin; /* smallest pooled origin index attaining num (P rows first); -1 if not computed   */
} ddks_result;

/* NCCL bootstrap: rank 0 calls this, the harness broadcasts the 128 bytes (e.g. via torch.distributed),
 * and every rank passes them to ddks_create. */
DDKS_API ddks_status ddks_get_nccl_id(void* out_128_bytes);

/* Create a context on CUDA device `device`. world >= 1, 0 <= rank < world. nccl_id must be NULL iff world == 1.
 * *out receives the context (NULL on failure). */
DDKS_API ddks_status ddks_create(ddks_ctx** out, int device, int world, int rank, const void* nccl_id, uint32_t flags);

/* Exact ddKS of one pair. P: [n_P][d], Q: [n_Q][d] (device or host). out: host. */
DDKS_API ddks_status ddks_stat(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                      void* stream, ddks_result* out);

/* B independent pairs (north_star (2); the power-analysis repeats of P:L364-371).
 * P: [B][n_P][d], Q: [B][n_Q][d] (device or host). out: host [B]; argmax_origin is -1 for batch items. */
DDKS_API ddks_status ddks_stat_batch(ddks_ctx* ctx, const float* P, const float* Q, int64_t B, int64_t n_P, int64_t n_Q,
                            int32_t d, void* stream, ddks_result* out);

/* Permutation null. pooled: [n_P+n_Q][d] (device or host), first n_P rows = P.
 * perms: [n_perm][n_P+n_Q] int32 (device or host); permutation j assigns pooled[perms[j][0..n_P)] to P' and
 * the rest to Q'; every row must be a permutation of 0..n_P+n_Q-1 (checked: DDKS_ERR_INVALID_ARGUMENT).
 * Outputs (host): null_num[n_perm]; *observed = the identity split; *p_value = (1 + #{null_num >= observed.num})
 * / (1 + n_perm). Any of null_num / observed / p_value may be NULL if not wanted. */
DDKS_API ddks_status ddks_permutation_null(ddks_ctx* ctx, const float* pooled, int64_t n_P, int64_t n_Q, int32_t d,
                                  const int32_t* perms, int64_t n_perm, void* stream, uint64_t* null_num,
                                  ddks_result* observed, double* p_value);

/* Debug / sampled-parity export: num(o) = max_q |c_P[q]*n_Q - c_Q[q]*n_P| for pooled origins [o_begin, o_end).
 * num_out: [o_end - o_begin] uint64, device or host. Single-rank (no collective). */
DDKS_API ddks_status ddks_stat_per_origin(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                                 int64_t o_begin, int64_t o_end, uint64_t* num_out, void* stream);

/* ---- Analytic significance (§3) ----------------------------------
 *   M_T[i,k] = # points of Q ("T") in orthant i about pooled test point k (all N pooled points),
 *   lambda   = (M_T[i,k] + 1) / (n_Q + 2)                            (Bayes estimator, uniform prior),
 *   p(d<=D)  = sum over (n_P', n_Q') in 0..n_P x 0..n_Q with |n_P' n_Q - n_Q' n_P| <= num
 *              of pmf(n_P' : n_P, lambda) pmf(n_Q' : n_Q, lambda)     ("<=" per DESIGN.md R12),
 *              pmf binomial, or Poisson with mean m*lambda if sig_flags has DDKS_SIG_POISSON,
 *   S        = 1 - prod over the 2^d orthants i and N test points k of p(d<=D)          (R13).
 * The statistic itself (out->stat) is computed exactly as ddks_stat does (same num/den/D/argmax).
 * log_prod = sum of log p(d<=D) over the 2^d N cells (each term computed as log1p(-(1 - p)), the complement summed
 * directly; R14); S = -expm1(log_prod). Terms of a pmf below e^-100 of its mode are omitted (absolute
 * error <= N e^-100 per cell).
 * Optional host/device outputs (NULL if not wanted): mt_hist[n_Q + 1] = number of cells with M_T = m;
 * log_p_table[n_Q + 1] = log p(d<=D | lambda_m) for every m with mt_hist[m] > 0, 0 elsewhere.
 * Multi-GPU: origins sharded as in ddks_stat; the histogram is all-reduced (sum) and the table entries are sharded;
 * every rank returns the full result. */
#define DDKS_SIG_POISSON 1u

typedef struct {
    ddks_result stat; /* the ddKS statistic (as ddks_stat) */
    double S;         /* significance: 1 - prod p(d <= D) (small S: reject "same distribution")  */
    double log_prod;  /* sum over the cells of log p(d <= D) (<= 0)                              */
    int64_t cells;    /* 2^d * (n_P + n_Q)                                                         */
} ddks_significance_result;

DDKS_API ddks_status ddks_significance(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                              uint32_t sig_flags, void* stream, ddks_significance_result* out, uint64_t* mt_hist,
                              double* log_p_table);

/* Batched significance: B independent pairs P[B][n_P][d], Q[B][n_Q][d] (device or host), each exactly as
 * ddks_significance (no histogram/table outputs); out: host [B], stat.argmax_origin = -1. Multi-GPU: items sharded,
 * every rank returns all B results. For the paper's repeated small tests (power analyses). */
DDKS_API ddks_status ddks_significance_batch(ddks_ctx* ctx, const float* P, const float* Q, int64_t B, int64_t n_P,
                                             int64_t n_Q, int32_t d, uint32_t sig_flags, void* stream,
                                             ddks_significance_result* out);

/* ---- vdKS: voxel approximation (§2.2.2, Alg. 1) -------------------
 * NormalizeData: per dimension over the pooled points, x' = (x - min)/(max - min) in double (a constant dimension
 * maps to 0.5; R15); IndexFromPoint: cell c_m = min(floor(x'_m k), k-1), k voxels per dimension;
 * Diff = VoxelList[Q]/n_Q - VoxelList[P]/n_P; for every filled voxel, the 2^d orthant sums of Diff split at the
 * voxel's lower corner (the voxel itself in the all->= orthant, as Eq. 3 places the origin; R16);
 * out->num = max over filled voxels and orthants of |sum| x n_P n_Q (exact integer), out->den = n_P n_Q,
 * out->D = num / den; out->argmax_origin = -1. k >= 1 and k^d <= 2^30 (else DDKS_ERR_TOO_LARGE).
 * Multi-GPU: points sharded for the voxel histogram (all-reduce sum), voxels sharded for the orthant sums. */
DDKS_API ddks_status ddks_vdks(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                               int64_t k, void* stream, ddks_result* out);

/* ---- rdKS: radial approximation (§2.2.3, Alg. 2) ------------------
 * NormalizeData as ddks_vdks; corners = the origin and the d unit axis vectors of the normalised space;
 * for each corner, Euclidean distances sqrt(sum_m (x'_m - c_m)^2) (f64, summed m = 0..d-1, correctly rounded sqrt)
 * of both samples, sorted, and GetDFromCornerLists = max over distinct distances r of
 * |#P(dist <= r) n_Q - #Q(dist <= r) n_P| (R17); out->num = the max over corners, out->den = n_P n_Q,
 * out->D = num / den, out->argmax_origin = the smallest CORNER index attaining num (0 = origin, m + 1 = e_m).
 * Any d >= 1 (the paper's high-d use: d = 1000); N (d + 1) < 2^34. Multi-GPU: corners sharded across ranks. */
DDKS_API ddks_status ddks_rdks(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                               void* stream, ddks_result* out);

/* Multi-GPU rehearsal on one device (scaling projections and shard-logic tests): ddks_stat restricted to the origin
 * shard that rank `rank` of `world` would own (same kernels, same shard — the strided origin blocks of the kd order
 * when the kd-ordered count runs — and no collective). out->num is the shard's maximum and out->argmax_origin the smallest pooled origin
 * attaining it; the max of the `world` nums, and the smallest argmax among the shards attaining that max, are
 * ddks_stat's result. ctx must be single-rank (world == 1 at ddks_create). */
DDKS_API ddks_status ddks_stat_shard(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                                     int world, int rank, void* stream, ddks_result* out);

/* Host-only helper (no GPU needed): the contiguous origin / item range [*begin, *end) that `rank` of `world`
 * owns out of `total` units. Ranges are balanced to within one unit and cover 0..total exactly. */
DDKS_API ddks_status ddks_shard_range(int64_t total, int world, int rank, int64_t* begin, int64_t* end);

/* ---- Multi-GPU combine steps (host-only, no GPU needed; the library calls them after its one all-gather, and they
 * are exported so the combine logic can be tested and reused with any transport, e.g. torch.distributed gloo) ---- */
typedef struct {
    uint64_t num;          /* this rank's max num(o) over its origin shard (0 if the shard is empty)            */
    int64_t argmax_origin; /* smallest pooled origin of the shard attaining num; -1 if none                     */
    uint32_t flags;        /* bit 0: non-finite input, bit 1: bad permutation row                              */
    uint32_t reserved;
} ddks_rank_record;

/* Combine the `world` per-rank records of one statistic (the max over the union of the origin shards):
 * out->num = max num; out->argmax_origin = the smallest argmax among the records attaining it (-1 if none);
 * out->flags = OR of the flags. recs: host [world]. */
DDKS_API ddks_status ddks_combine_records(const ddks_rank_record* recs, int world, ddks_rank_record* out);

/* Unpad the all-gathered per-item block of a sharded batch / permutation / batched-significance call. Layout: world
 * records of stride = n_arr * chunk + 1 uint64, chunk = ceil(total / world) (rank 0's shard, the largest); record r
 * holds rank r's slice ddks_shard_range(total, world, r) of each of the n_arr arrays, each padded to chunk, then
 * rank r's flags word. out: host [n_arr][total]; *flags (may be NULL) = OR of the ranks' flags. */
DDKS_API ddks_status ddks_unpad_items(const uint64_t* gathered, int64_t total, int world, int n_arr, uint64_t* out,
                                      uint32_t* flags);

/* Number of kernels the library launched on this context since creation (for the bench's gpu_launches). */
DDKS_API int64_t ddks_launch_count(const ddks_ctx* ctx);

/* Levels K of the kd ordering used by the last count on this context (0: position order, no bit elision;
 * K >= 1: bits 0..K-1 decided per tile where possible). Host-only, for tests and the bench line. */
DDKS_API int32_t ddks_kd_levels(const ddks_ctx* ctx);

/* 1 if the last count on this context was the rank-lane count (position order: each pair's d compares are
 * ceil(d/3) 32-bit integer adds on 10-bit per-CTA rank lanes; DESIGN.md §7 "rank lanes"), else 0. Host-only. */
DDKS_API int32_t ddks_rank_lanes(const ddks_ctx* ctx);

/* Profiling (context created with DDKS_FLAG_PROFILE): totals since the last read, then reset.
 * count_ms: summed device time of the classify+count kernel launches (CUDA events on the call's stream);
 * launches: how many such launches; pairs: point-pair orthant classifications they performed (sum of
 * items x origins x points; for the label-invariant permutation kernel, one classification per pair per chunk of
 * permutations it serves); any pointer may be NULL. */
DDKS_API ddks_status ddks_profile_read(ddks_ctx* ctx, double* count_ms, int64_t* launches, uint64_t* pairs);

/* In-kernel clock probe (context created with DDKS_FLAG_PROFILE): one lane per count-kernel CTA reads clock64 and
 * %globaltimer around its classify+count loop; *sm_mhz = summed SM cycles / summed ns over those CTAs since the last
 * read (0 if none), i.e. the SM clock the counting actually ran at. Resets the totals. */
DDKS_API ddks_status ddks_profile_clock(ddks_ctx* ctx, double* sm_mhz);

/* Executed work of the count kernels (context created with DDKS_FLAG_PROFILE), totals since the last read, then reset:
 * *compares = FP32 orthant compares the classify kernels actually executed (every lane of every warp, clamped tail
 * slots included; the bits the kd / warp-level orderings decide once per tile or sub-tile are not compares). The
 * method's algorithmic work is d compares per pair classification; with the kd ordering the executed count is lower.
 * Counted in-kernel (one add per warp and tile), so it tracks whichever kernel variant ran. */
DDKS_API ddks_status ddks_profile_work(ddks_ctx* ctx, uint64_t* compares);

/* Destroy a context (NULL-safe). Frees workspace and the NCCL communicator. */
DDKS_API ddks_status ddks_destroy(ddks_ctx* ctx);

/* Last error message of this context ("" if none); valid until the next call on ctx. ctx may be NULL
 * (then the message of the last failed ddks_create on this thread). */
DDKS_API const char* ddks_last_error(const ddks_ctx* ctx);

/* Library version string. */
DDKS_API const char* ddks_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DDKS_H_ */
