// ddks_significance.cuh — analytic significance S of a ddKS statistic (§3).
//
//   M_T[i,k]  = # points of T (= Q) in orthant i about pooled test point k
//   lambda    = (M_T[i,k] + 1) / (N_T + 2)                                              (Bayes estimator)
//   p(n:m,l)  = C(m,n) l^n (1-l)^(m-n)        or the Poisson pmf e^{-ml}(ml)^n/n!
//   p(d<=D)   = sum over the Delta band |n_P N_T - n_T N_P| <= num of p(n_P:N_P,l) p(n_T:N_T,l)
//   S         = 1 - prod over the 2^d x N cells of p(d<=D)
//
// B200 design (DESIGN.md §7 "significance"):
//   * the classify+count pass runs in SPLIT mode (c_P, c_Q kept apart) and its finaliser also histograms the
//     M_T values: hist[m] = #cells with M_T = m. A cell's factor depends only on m, so the product becomes
//     sum_m hist[m] * log p(d<=D | lambda_m): at most N_T + 1 table entries instead of 2^d N cells;
//   * k_sig_table: one persistent CTA per table entry in flight. It evaluates the pmf of n_P over the window
//     where it is within e^-100 of its mode (warp-parallel 32-ary searches on the unimodal log pmf), prefix- and
//     suffix-scans it
//     in global scratch, and sums the COMPLEMENT q = 1 - p(d<=D) = sum_{n_T} p(n_T) [F_P(lo-1) + (1 - F_P(hi))]
//     (only tail sums of small positive terms: no cancellation). log p(d<=D) = log1p(-q) (R14);
//   * log n! comes from a device table LF[n] = lgamma(n+1);
//   * the sum over the table is a fixed-order block reduction (deterministic run to run).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"

namespace ddks {

__global__ void k_logfact(double* __restrict__ LF, int64_t n_max) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_max; i += (int64_t)gridDim.x * blockDim.x)
        LF[i] = lgamma((double)i + 1.0);
}

struct SigArgs {
    const double* LF;                    // [lf_max + 1] log n!
    int64_t lf_max;                      // >= max(N_P, N_T); Poisson: room for the pmf mass beyond N
    const unsigned long long* hist;      // [B][N_T + 1] cells with M_T = m (all ranks' cells), per item
    const unsigned long long* num;       // device [B]: the items' statistic numerators (after any all-reduce)
    int64_t N_P, N_T;
    int64_t m_begin, m_end;              // flat table entries e = item * (N_T + 1) + m this rank evaluates
    int poisson;
    double* scratch;                     // [gridDim.x][2][W_max]
    int64_t W_max;
    double* table;                       // [B][N_T + 1] log p(d <= D | lambda_m); 0 where hist[m] == 0
    double* contrib;                     // [B][N_T + 1] hist[m] * table[m]
    uint32_t* flag;                      // |= 4 if a window exceeded W_max (host retries with a larger W_max)
};

// log p(n : m, lambda) (binomial) or log Poisson(n ; m lambda)
struct LogPmf {
    const double* LF;
    int64_t m;
    double loglam, log1m, mu, logmu;
    int poisson;
    __device__ __forceinline__ void init(const double* LF_, int64_t m_, double lam, int poisson_) {
        LF = LF_;
        m = m_;
        poisson = poisson_;
        loglam = log(lam);
        log1m = log1p(-lam);
        mu = (double)m_ * lam;
        logmu = log(mu);
    }
    __device__ __forceinline__ double operator()(int64_t n) const {
        DDKS_ASSERT(n >= 0);
        if (poisson) return -mu + (double)n * logmu - LF[n];
        return LF[m] - LF[n] - LF[m - n] + (double)n * loglam + (double)(m - n) * log1m;
    }
    __device__ __forceinline__ int64_t mode(double lam) const {
        int64_t k = poisson ? (int64_t)floor(mu) : (int64_t)floor((double)(m + 1) * lam);
        return k < 0 ? 0 : (k > m ? m : k);
    }
    // Warp-cooperative 32-ary searches (all 32 lanes call them; every lane gets the result).
    // Largest n in [lo, hi] with f(n) >= thr, f non-increasing there and f(lo) >= thr.
    __device__ int64_t warp_last_above(int64_t lo, int64_t hi, double thr) const {
        const int lane = threadIdx.x & 31;
        while (hi - lo > 31) {
            const int64_t step = (hi - lo) / 31 + 1;  // 31 steps reach past hi
            const int64_t c = lo + lane * step;
            const uint32_t ok = __ballot_sync(0xffffffffu, c <= hi && (*this)(c) >= thr);  // a prefix of lanes
            const int k = 31 - __clz(ok);
            lo = lo + k * step;
            hi = min(hi, lo + step - 1);
        }
        const int64_t c = lo + lane;
        const uint32_t ok = __ballot_sync(0xffffffffu, c <= hi && (*this)(c) >= thr);
        return lo + (31 - __clz(ok));
    }
    // Smallest n in [lo, hi] with f(n) >= thr, f non-decreasing there and f(hi) >= thr.
    __device__ int64_t warp_first_above(int64_t lo, int64_t hi, double thr) const {
        const int lane = threadIdx.x & 31;
        while (hi - lo > 31) {
            const int64_t step = (hi - lo) / 31 + 1;  // 31 steps reach past hi
            const int64_t c = hi - lane * step;
            const uint32_t ok = __ballot_sync(0xffffffffu, c >= lo && (*this)(c) >= thr);  // a prefix of lanes
            const int k = 31 - __clz(ok);
            hi = hi - k * step;
            lo = max(lo, hi - step + 1);
        }
        const int64_t c = hi - lane;
        const uint32_t ok = __ballot_sync(0xffffffffu, c >= lo && (*this)(c) >= thr);
        return hi - (31 - __clz(ok));
    }
    // [a, b] = the n in 0..m with log pmf >= log pmf(mode) - 100 (the pmf is unimodal). Poisson only: [ta, tb] =
    // the n > m (outside the Delta set's 0..m) above the same threshold, tb <= lf_max; ta > tb if there are none.
    // Called by a whole warp.
    __device__ void window(double lam, int64_t lf_max, int64_t& a, int64_t& b, int64_t& ta, int64_t& tb) const {
        const int64_t md = mode(lam);
        const double thr = (*this)(md) - 100.0;
        a = warp_first_above(0, md, thr);
        b = warp_last_above(md, m, thr);
        ta = m + 1;
        tb = m;
        if (poisson && m < lf_max && (*this)(m + 1) >= thr) tb = warp_last_above(m + 1, lf_max, thr);
    }
};

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];  // same order in every thread
    return s;
}

// In-place inclusive scan of x[0..W) (REV: from the right, x[i] = sum_{j >= i}). Fixed order: chunks of NT
// consecutive elements, one per thread (coalesced), each chunk scanned with warp shuffles + a scan of the warp
// totals, plus the running carry of the earlier chunks.
template <int NT, bool REV>
__device__ void block_scan(double* x, int64_t W, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double carry = 0.0;
    for (int64_t base = 0; base < W; base += NT) {
        const int64_t i = base + threadIdx.x;
        const int64_t j = REV ? W - 1 - i : i;
        double v = i < W ? x[j] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) red[w] = v;
        __syncthreads();
        if (w == 0) {
            double t = lane < NT / 32 ? red[lane] : 0.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            if (lane < NT / 32) red[lane] = t;  // inclusive prefix of the warp totals
        }
        __syncthreads();
        const double before = carry + (w ? red[w - 1] : 0.0);
        if (i < W) x[j] = before + v;
        carry += red[NT / 32 - 1];
        __syncthreads();  // red is rewritten by the next chunk
    }
}

// floor(x / n) and ceil(x / n) for n > 0, exact: a double-precision estimate (inv = 1/n) corrected by the integer
// remainder (64-bit integer division is a long emulated sequence on the GPU; this is two FMAs and a check).
__device__ __forceinline__ int64_t floor_div(int64_t x, int64_t n, double inv) {
    int64_t q = (int64_t)floor((double)x * inv);
    int64_t r = x - q * n;
    while (r < 0) { --q; r += n; }
    while (r >= n) { ++q; r -= n; }
    return q;
}
__device__ __forceinline__ int64_t ceil_div(int64_t x, int64_t n, double inv) { return -floor_div(-x, n, inv); }

constexpr int SIG_T = 512;

__global__ void __launch_bounds__(SIG_T) k_sig_table(const SigArgs a) {
    __shared__ double red[SIG_T];
    __shared__ int64_t win[8];
    double* A = a.scratch + (int64_t)blockIdx.x * 2 * a.W_max;  // inclusive prefix sums of p(n_P)
    double* B = A + a.W_max;                                     // inclusive suffix sums of p(n_P)
    const double invT = 1.0 / (double)a.N_T;
    for (int64_t e = a.m_begin + blockIdx.x; e < a.m_end; e += gridDim.x) {
        const int64_t item = e / (a.N_T + 1), m = e - item * (a.N_T + 1);
        const int64_t num = (int64_t)a.num[item];
        const unsigned long long h = a.hist[e];
        if (h == 0) {
            if (threadIdx.x == 0) a.table[e] = 0.0, a.contrib[e] = 0.0;
            continue;
        }
        const double lam = ((double)m + 1.0) / ((double)a.N_T + 2.0);
        LogPmf fP, fT;
        fP.init(a.LF, a.N_P, lam, a.poisson);
        fT.init(a.LF, a.N_T, lam, a.poisson);
        if (threadIdx.x < 32) {  // warp 0: the n_P window, warp 1: the n_T window
            int64_t w0, w1, w2, w3;
            fP.window(lam, a.lf_max, w0, w1, w2, w3);
            if (threadIdx.x == 0) win[0] = w0, win[1] = w1, win[4] = w2, win[5] = w3;
        } else if (threadIdx.x < 64) {
            int64_t w0, w1, w2, w3;
            fT.window(lam, a.lf_max, w0, w1, w2, w3);
            if (threadIdx.x == 32) win[2] = w0, win[3] = w1, win[6] = w2, win[7] = w3;
        }
        __syncthreads();
        const int64_t aP = win[0], bP = win[1], aT = win[2], bT = win[3];
        int64_t W = bP - aP + 1;
        if (W > a.W_max || (a.poisson && (win[5] == a.lf_max || win[7] == a.lf_max))) {
            if (threadIdx.x == 0) atomicOr(a.flag, 4u);
            W = W > a.W_max ? a.W_max : W;
        }
        // Poisson: the pmf restricted to the Delta set's 0..N has mass Z = 1 - t < 1, so the band sum p(d<=D)
        // (P:L255-268 with the Poisson pmf, R12) is Z_P Z_T - (mass outside the band), and
        // 1 - p = t_P + t_T - t_P t_T + (mass outside the band); t = the Poisson mass beyond N, summed directly
        double tP = 0.0, tT = 0.0;
        if (a.poisson) {
            double sP = 0.0, sT = 0.0;
            for (int64_t n = win[4] + threadIdx.x; n <= win[5]; n += SIG_T) sP += exp(fP(n));
            for (int64_t n = win[6] + threadIdx.x; n <= win[7]; n += SIG_T) sT += exp(fT(n));
            tP = block_sum<SIG_T>(sP, red);
            tT = block_sum<SIG_T>(sT, red);
        }
        const int64_t eP = aP + W - 1;  // last n_P inside the window
        // lo(n_T) and hi(n_T) increase with n_T: if the band covers the whole n_P window already at the ends of the
        // n_T window, every tail below is exactly 0 and the pmf tables are not needed (the usual case when D is
        // many standard deviations above the sampling noise)
        const bool covered = ceil_div(bT * a.N_P - num, a.N_T, invT) <= aP && floor_div(aT * a.N_P + num, a.N_T, invT) >= eP;
        if (!covered) {
            for (int64_t i = threadIdx.x; i < W; i += SIG_T) {
                const double v = exp(fP(aP + i));
                A[i] = v;
                B[i] = v;
            }
            __syncthreads();
            block_scan<SIG_T, false>(A, W, red);
            block_scan<SIG_T, true>(B, W, red);
        }
        double acc = 0.0;
        for (int64_t nT = aT + threadIdx.x; !covered && nT <= bT; nT += SIG_T) {
            // band of n_P with |n_P N_T - nT N_P| <= num: [lo, hi], exact int64
            const int64_t lo = ceil_div(nT * a.N_P - num, a.N_T, invT);
            const int64_t hi = floor_div(nT * a.N_P + num, a.N_T, invT);
            DDKS_ASSERT(lo <= aP || (lo > eP + 1 ? eP + 1 : lo) - 1 - aP < W);
            DDKS_ASSERT(hi >= eP || (hi < aP - 1 ? aP - 1 : hi) + 1 - aP >= 0);
            const double left = lo <= aP ? 0.0 : A[(lo > eP + 1 ? eP + 1 : lo) - 1 - aP];   // sum_{n_P < lo}
            const double right = hi >= eP ? 0.0 : B[(hi < aP - 1 ? aP - 1 : hi) + 1 - aP];  // sum_{n_P > hi}
            const double tail = left + right;
            if (tail != 0.0) acc += exp(fT(nT)) * tail;
        }
        const double q = block_sum<SIG_T>(acc, red) + (tP + tT - tP * tT);
        if (threadIdx.x == 0) {
            const double lp = log1p(-q);
            a.table[e] = lp;
            a.contrib[e] = (double)h * lp;
        }
        __syncthreads();  // scratch and win reused by the next entry
    }
}

// Fixed-order sum of contrib[b..e) -> *out (one CTA); batch: CTA i sums [b + i*stride, e + i*stride) -> out[i].
__global__ void __launch_bounds__(SIG_T) k_sig_sum(const double* __restrict__ contrib, int64_t b, int64_t e,
                                                   double* out, int64_t stride = 0) {
    __shared__ double red[SIG_T];
    contrib += blockIdx.x * stride;
    out += blockIdx.x;
    const int64_t n = e - b;
    const int64_t C = (n + SIG_T - 1) / SIG_T;
    const int64_t lo = b + threadIdx.x * C, hi = lo + C < e ? lo + C : e;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += contrib[i];
    s = block_sum<SIG_T>(s, red);
    if (threadIdx.x == 0) *out = s;
}

}  // namespace ddks
