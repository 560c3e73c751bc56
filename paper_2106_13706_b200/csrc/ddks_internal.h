// ddks_internal.h — host-side internals shared by the translation units of libddks.so (NOT part of the C ABI):
// the context, device workspace buffers, error macros and the helpers the C-ABI entry points are built from.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ddks.h"
#include "ddks_common.cuh"

constexpr int kMaxDevices = 64;  // per-device, per-kernel launch attributes are cached for this many devices

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// Device-side result block of one statistic on one rank (one D2H per call; with world > 1 it is also the 32-byte record
// every rank contributes to the single all-gather of ddks_stat, combined on the host by ddks_combine_records).
struct DevResult {
    unsigned long long num;  // max num(o) over this rank's origins
    unsigned long long arg;  // smallest pooled origin attaining it (~0: none / not computed; k_argmax path)
    unsigned long long key;  // packed argmax (num / gcd) << 31 | (2^31 - 1 - origin) (0: none; fused path)
    uint32_t flag;           // bit 0: non-finite input, bit 1: bad permutation row, bit 2: significance scratch
    uint32_t pad;
};
static_assert(sizeof(DevResult) == 32, "DevResult is the 32-byte all-gather record");

struct ddks_ctx {
    int device = 0, world = 1, rank = 0;
    uint32_t flags = 0;
    ncclComm_t comm = nullptr;
    DevBuf raw_a, raw_b, raw_perm, packed, packed2, pool_packed, per_origin, accum, item_num, bitmap, labels, res;
    DevBuf gather;  // world > 1: all-gather send + receive buffers
    DevBuf sig_hist, sig_lf, sig_scratch, sig_table, sig_contrib, sig_part;  // ddks_significance workspace
    DevBuf vox_keys, vox_cnt, vox_S, vox_fill, vox_slab;                      // ddks_vdks workspace
    void* vox_zero_p = nullptr;  // vox_cnt.p whose first vox_zero bytes are known zero (slab scans clean the counts)
    size_t vox_zero = 0;
    DevBuf rd_keys, rd_xn, rd_k0, rd_k1, rd_hist, rd_tcnt, rd_cnum;              // ddks_rdks workspace
    DevBuf x0_keys0, x0_keys1, x0_hist, x0_pts, x0_perm, x0_pts2, x0_perm2, x0_boxes;  // kd-ordered count workspace
    DevBuf rdb_cnt, rdb_pst, rdb_coff, rdb_fill, rdb_clist, rdb_csum, rdb_bits;  // rdKS bucket-pruned sweep
    DevBuf rank_v;            // rank-lane count: V_k of every origin block in Eytzinger order (ddks_rank.cuh)
    DevBuf kdf_bar, kdf_buf;  // fused mid-N kd ordering (k_kdb_fused): grid barrier; ranges, chunk totals, histograms
    void* rdb_zero_p = nullptr;  // rdb_cnt.p whose first rdb_zero bytes are known zero (the sweep re-zeroes the counts)
    size_t rdb_zero = 0;
    DevBuf prof_clk;  // [3] u64: SM cycles, globaltimer ns, executed compares summed over count CTAs (DDKS_FLAG_PROFILE)
    void* host_pinned = nullptr;  // DevResult + scratch
    size_t host_pinned_bytes = 0;
    int64_t launches = 0;
    int kd_levels = 0;  // levels of the last kd-ordered count (0: position order)
    int rank_lanes = 0;  // the last count was the rank-lane count (ddks_rank.cuh)
    std::string err;
    // profiling (DDKS_FLAG_PROFILE)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending, ev_free;
    std::vector<uint64_t> ev_pairs;
    std::vector<char> ev_recycle;  // parallel to ev_pending: return the pair to ev_free (0: owned by a CUDA graph)
    // ddks_stat CUDA graph (DESIGN.md §7 "graphs"): the whole call -- H2D of pinned inputs, pack, count, finalise,
    // argmax, collectives, D2H -- captured on the second identical call and replayed by one cudaGraphLaunch after
    uint64_t alloc_epoch = 0;  // bumped on every workspace (re)allocation: a captured graph holds raw pointers
    struct StatKey {
        const void *P = nullptr, *Q = nullptr;
        int64_t n_P = -1, n_Q = -1;
        int d = 0;
        uint64_t epoch = ~0ull;
        bool operator==(const StatKey& o) const {
            return P == o.P && Q == o.Q && n_P == o.n_P && n_Q == o.n_Q && d == o.d && epoch == o.epoch;
        }
    };
    StatKey sg_seen, sg_key;
    cudaGraphExec_t sg_exec = nullptr;
    cudaStream_t cap_stream = nullptr;
    // host-input batches: H2D copies of item chunks on copy_stream, overlapped with the counts of earlier chunks
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> copy_evs;
    int64_t sg_launches = 0;
    int sg_kd_levels = 0, sg_rank_lanes = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> sg_evs;
    std::vector<uint64_t> sg_ev_pairs;
    // the same for ddks_stat_batch and ddks_permutation_null (run_call in ddks_api.cu): key = the call's pointers,
    // sizes, flags and the workspace epoch; captured on the second identical call, replayed from the third
    struct CallGraph {
        std::vector<uint64_t> seen, key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
        std::vector<uint64_t> ev_pairs;
    };
    CallGraph cg_batch, cg_null, cg_vdks, cg_rdks;
    double prof_ms = 0.0;
    int64_t prof_launches = 0;
    uint64_t prof_pairs = 0;
};

extern thread_local std::string g_create_err;

namespace ddks_host {

ddks_status fail(ddks_ctx* c, ddks_status s, const char* fmt, ...);

#define CU(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? DDKS_ERR_OOM : DDKS_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
    } while (0)

#define NC(call)                                                                                         \
    do {                                                                                                 \
        ncclResult_t r_ = (call);                                                                        \
        if (r_ != ncclSuccess)                                                                           \
            return fail(ctx, DDKS_ERR_NCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
    } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())

// Profiling event record: under stream capture it must be an external record node (a plain record is only a
// dependency marker there and cannot be timed); outside capture the external flag is refused.
inline cudaError_t record_event(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t r = cudaStreamIsCapturing(st, &cs);
    if (r != cudaSuccess) return r;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                               : cudaEventRecord(e, st);
}

// DDKS_FLAG_PROFILE: an event pair around the dominant launch of a call (no-op without the flag); prof_end queues it
// with its work units (pair classifications, or REDs for the approximations) for collect_profile after the sync
ddks_status prof_begin(ddks_ctx* ctx, cudaStream_t st, std::pair<cudaEvent_t, cudaEvent_t>* ev);
ddks_status prof_end(ddks_ctx* ctx, cudaStream_t st, const std::pair<cudaEvent_t, cudaEvent_t>& ev, uint64_t units);
ddks_status collect_profile(ddks_ctx* ctx);

// grow-only device workspace; host (pinned) scratch
ddks_status ensure(ddks_ctx* ctx, DevBuf& b, size_t bytes);
// as ensure, and a (re)allocated buffer is zeroed on st (buffers whose users leave them zero: count partials)
ddks_status ensure_zeroed(ddks_ctx* ctx, DevBuf& b, size_t bytes, cudaStream_t st);
// the profiling counters (DDKS_FLAG_PROFILE): prof_clk allocated and zeroed once
ddks_status ensure_prof(ddks_ctx* ctx);
ddks_status ensure_host(ddks_ctx* ctx, size_t bytes);
// device pointers are used in place, host pointers copied on st into buf
ddks_status stage_input(ddks_ctx* ctx, const void* src, size_t bytes, DevBuf& buf, cudaStream_t st, const void** out);
uint64_t gcd_u64(uint64_t a, uint64_t b);
ddks_status check_sizes(ddks_ctx* ctx, int64_t n_P, int64_t n_Q, int32_t d);
int pad_dim(int d);
ddks_status bind_device(ddks_ctx* ctx);
ddks_status collect_profile(ddks_ctx* ctx);
// validate (NaN/Inf -> *flag |= 1) and pack P then Q into [B][N][pad_dim(d)] rows
ddks_status launch_pack(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t B,
                        float* dst, uint32_t* flag, cudaStream_t st);
// batches: near-x_0-sorted pack of every label run when the items are small (*wx: the count may use k_count<WX>)
ddks_status launch_pack_batch(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d,
                              int64_t B, float* dst, uint32_t* flag, cudaStream_t st, bool* wx);
// one statistic over the origin shard [ob, oe): count + this rank's argmax candidate, no collective unless
// reduce_num_first (see ddks_api.cu); (kd order: the strided origin blocks of shard sr of sw instead of [ob, oe))
ddks_status count_statistic(ddks_ctx* ctx, const float* packed, int d, int64_t n_P, int64_t n_Q, int64_t ob,
                            int64_t oe, int sw, int sr, DevResult* dres, bool export_per, bool split,
                            unsigned long long* hist, cudaStream_t st, uint64_t** per_out, bool reduce_num_first);
// the fused packed-key argmax applies (n_P n_Q / gcd < 2^33)
bool argmax_key_fits(int64_t n_P, int64_t n_Q);
// a rank's device result -> host record (decodes the packed key when use_key)
ddks_rank_record decode_record(const DevResult& r, int64_t n_P, int64_t n_Q, bool use_key);
// B items of N packed points: classify + count (+ finalise); force_split + hist: SPLIT counters and per-item M_T
// histograms hist[B][n_Q + 1] (significance); best_key (B == 1): the fused packed argmax
ddks_status run_count(ddks_ctx* ctx, const float* packed, int d, int64_t B, int64_t n_P, int64_t n_Q,
                      int64_t o_begin, int64_t o_end, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st,
                      bool force_split = false, unsigned long long* hist = nullptr, bool wx = false,
                      unsigned long long* best_key = nullptr);
// the rank-lane count (ddks_rank.cuh, ddks_api_rank.cu): one statistic (B == 1) at 2 <= d <= 8, >= convention,
// position order, origins [o_begin, o_end); DIFF counters, or SPLIT (c_P and c_Q apart, hist as run_count) in two
// launches over the P rows and the Q rows; results as run_count
ddks_status run_count_rank(ddks_ctx* ctx, const float* packed, int d, int64_t n_P, int64_t n_Q, int64_t o_begin,
                           int64_t o_end, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st,
                           unsigned long long* best_key, bool split = false, unsigned long long* hist = nullptr);
// items sharded contiguously over ranks: one all-gather of padded records (n_arr arrays + flags) into host hbuf
ddks_status gather_items(ddks_ctx* ctx, uint64_t* const* dev, int n_arr, int64_t total, const uint32_t* dflag,
                         cudaStream_t st, uint64_t* hbuf);
int64_t gather_stride(int64_t total, int world, int n_arr);
// kd-ordered count of one statistic (B == 1, 2 <= D <= 8; ddks_kd.cuh, instantiated in ddks_api_kd_*.cu): the origin
// blocks shard_rank, shard_rank + shard_world, ... of the kd order
template <int D>
ddks_status run_count_kd_d(ddks_ctx* ctx, const float* packed, int64_t n_P, int64_t n_Q, int shard_world,
                           int shard_rank, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st, bool split,
                           unsigned long long* hist, unsigned long long* best_key);
ddks_status radix_sort_keys(ddks_ctx* ctx, uint64_t* src, uint64_t* dst, int64_t N, int nseg, int shift_begin,
                            uint32_t* hist, cudaStream_t st, uint64_t** sorted);

// ---- per-call-shape CUDA graphs (ddks_api.cu) ------------------------------------------------------------------
bool graph_input_ok(const void* p);   // a graph may read p at replay time (device, managed or pinned host memory)
bool env_overrides();                 // a tuning / test environment knob is set: no graphs
void drop_call_graph(ddks_ctx* ctx, ddks_ctx::CallGraph& cg);
void launch_call_graph(ddks_ctx* ctx, ddks_ctx::CallGraph& cg, cudaStream_t st, cudaError_t* e);

// Run the stream-ordered part of a C-ABI call (enq: staging, kernels, collectives, the D2H into host_pinned; no sync)
// through a per-call-shape CUDA graph: the second call with the same key (pointers, sizes, flags, plan state; + the
// workspace epoch) is captured on the context's capture stream and every identical call after it is one
// cudaGraphLaunch on st. Not graphable (host inputs in pageable memory, DDKS_FLAG_NO_GRAPH, environment
// overrides): enq runs on st. Host-side state updates belong outside enq (a replay does not run it).
template <class F>
ddks_status run_call(ddks_ctx* ctx, ddks_ctx::CallGraph& cg, std::vector<uint64_t> key, bool graphable,
                     cudaStream_t st, F&& enq) {
    graphable = graphable && !(ctx->flags & DDKS_FLAG_NO_GRAPH) && !env_overrides();
    key.push_back(ctx->alloc_epoch);
    cudaError_t e;
    if (graphable && cg.exec && cg.key == key) {
        launch_call_graph(ctx, cg, st, &e);
        CU(e);
        return DDKS_OK;
    }
    if (graphable && cg.seen == key) {
        drop_call_graph(ctx, cg);
        if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        const size_t ev0 = ctx->ev_pending.size();
        const int64_t l0 = ctx->launches;
        CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
        const ddks_status s = enq(ctx->cap_stream);
        cudaGraph_t g = nullptr;
        e = cudaStreamEndCapture(ctx->cap_stream, &g);
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs(ctx->ev_pending.begin() + ev0, ctx->ev_pending.end());
        std::vector<uint64_t> pairs(ctx->ev_pairs.begin() + ev0, ctx->ev_pairs.end());
        ctx->ev_pending.resize(ev0);
        ctx->ev_pairs.resize(ev0);
        ctx->ev_recycle.resize(ev0);
        const int64_t nl = ctx->launches - l0;
        ctx->launches = l0;
        cudaGraphExec_t ex = nullptr;
        const bool good = s == DDKS_OK && e == cudaSuccess && g && ctx->alloc_epoch == key.back() &&
                          cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (good) {
            cg.exec = ex;
            cg.key = key;
            cg.launches = nl;
            cg.evs = evs;
            cg.ev_pairs = pairs;
            launch_call_graph(ctx, cg, st, &e);
            CU(e);
            return DDKS_OK;
        }
        cudaGetLastError();  // capture refused or the workspace moved: run uncaptured
        for (auto& v : evs) ctx->ev_free.push_back(v);
        ctx->err.clear();
    }
    ddks_status s = enq(st);
    if (s) return s;
    if (graphable) {  // a second identical call (same workspace) will be captured
        cg.seen = key;
        cg.seen.back() = ctx->alloc_epoch;
    }
    return DDKS_OK;
}

}  // namespace ddks_host
