/*
 * ddks_oracle.c — TEST INFRASTRUCTURE ONLY. Plain, slow, obviously-correct CPU oracle for the exact
 * ddKS statistic of arxiv 2106.13706. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or execute this file. The product path
 * (paper_2106_13706_b200/) never links or imports it, and it shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited as P:L<line>):
 *   - P:L33-35 (§2.1, Eq. 1): D = max |C_P(x) - C_T(x)|, C = orthant occupancy about x.
 *   - P:L40-44 (§2.1, Eq. 2): C evaluated at every point of both samples (pooled origins, P then T),
 *     maximum taken over the concatenation of both evaluation sets.
 *   - P:L46 (§2.1): "for each test point ... define each orthant ... determine the number of points
 *     from each sample that exist in that orthant" — the loop method, written out below as-is.
 *   - P:L59-67 (§2.2.1, Eq. 3): the comparison is element-wise "greater than or equal":
 *     bit k of the orthant code is [x_k >= o_k]  (reading R1: ties and the origin itself
 *     land on the >= side). ties_gt=1 switches to [x_k > o_k]; used only by tests to show the
 *     convention matters.
 *   - P:L68-75 (Eq. 4-5): the printed square-wave selector is degenerate; the orthant index is the
 *     binary code sum_k bit_k 2^k (reading R3; the numbering does not change D).
 *   - P:L78-81 (Eq. 6) and P:L238 (§3): per-sample normalised difference
 *     |c_P/n_P - c_T/n_T|, kept exact as the integer |c_P*n_T - c_T*n_P| over den = n_P*n_T
 *     (reading R2); D = (double)num / (double)den, one correctly rounded division (R5).
 *   - P:L371 (§4.2): permutation test; p = (1 + #{null >= observed}) / (1 + n_perm) (SPEC S:L363
 *     add-one convention; reading R9).
 *
 * Arithmetic: coordinates are read as float32 and compared after widening to double (exact and
 * order-preserving, so identical to an IEEE float32 ordered >=; -0 == +0; denormals compared
 * exactly). Counts are int64. No blocking, fusion or loop reordering: for each origin, for each
 * point, for each dimension — the paper's loop method. Origins are independent, so the outer loop
 * may run on several OpenMP threads (the integer max does not depend on order).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o libddks_oracle.so ddks_oracle.c   (no -ffast-math)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* P:L46 / P:L59-67: orthant code of `point` about `test_point` (SPEC S:L100-108 orthant_index). */
int oracle_orthant_index(const float* test_point, const float* point, int d, int ties_gt)
{
    int code = 0;
    for (int k = 0; k < d; ++k) {
        double x = (double)point[k];
        double o = (double)test_point[k];
        int bit = ties_gt ? (x > o) : (x >= o);
        code += bit << k;
    }
    return code;
}

/* SPEC S:L110-118 membership: counts[i][j] = #{points of `counted` in orthant j about test i}. */
void oracle_membership(const float* counted, int64_t n_counted, const float* test, int64_t n_test,
                       int d, int ties_gt, int64_t* counts /* [n_test][2^d] */)
{
    int64_t nq = (int64_t)1 << d;
    for (int64_t i = 0; i < n_test; ++i) {
        for (int64_t j = 0; j < nq; ++j) counts[i * nq + j] = 0;
        for (int64_t x = 0; x < n_counted; ++x) {
            int code = oracle_orthant_index(test + i * d, counted + x * d, d, ties_gt);
            counts[i * nq + code] += 1;
        }
    }
}

/* Pooled point i: rows of P first, then rows of Q (Eq. 2 concatenation order). */
static const float* pooled_row(const float* P, int64_t n_P, const float* Q, int d, int64_t i)
{
    return (i < n_P) ? (P + i * d) : (Q + (i - n_P) * d);
}

/* num(o) for one origin: max over orthants q of |cP[q]*n_Q - cQ[q]*n_P|. */
static uint64_t origin_num(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d,
                           int ties_gt, const float* origin, int64_t* cP, int64_t* cQ)
{
    int64_t nq = (int64_t)1 << d;
    for (int64_t q = 0; q < nq; ++q) { cP[q] = 0; cQ[q] = 0; }
    for (int64_t x = 0; x < n_P; ++x) cP[oracle_orthant_index(origin, P + x * d, d, ties_gt)] += 1;
    for (int64_t x = 0; x < n_Q; ++x) cQ[oracle_orthant_index(origin, Q + x * d, d, ties_gt)] += 1;
    uint64_t best = 0;
    for (int64_t q = 0; q < nq; ++q) {
        int64_t diff = cP[q] * n_Q - cQ[q] * n_P;
        uint64_t a = (uint64_t)(diff < 0 ? -diff : diff);
        if (a > best) best = a;
    }
    return best;
}

/* Per-origin num(o) for pooled origins [o_begin, o_end). out[o - o_begin]. Returns 0 on success. */
int oracle_ddks_per_origin(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int ties_gt,
                           int64_t o_begin, int64_t o_end, uint64_t* out, int nthreads)
{
    if (d < 1 || d > 20 || n_P < 1 || n_Q < 1 || o_begin < 0 || o_end > n_P + n_Q || o_begin > o_end) return 1;
    int64_t nq = (int64_t)1 << d;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        int64_t* cP = (int64_t*)malloc(sizeof(int64_t) * nq);
        int64_t* cQ = (int64_t*)malloc(sizeof(int64_t) * nq);
#pragma omp for schedule(dynamic, 16)
        for (int64_t o = o_begin; o < o_end; ++o)
            out[o - o_begin] = origin_num(P, n_P, Q, n_Q, d, ties_gt, pooled_row(P, n_P, Q, d, o), cP, cQ);
        free(cP);
        free(cQ);
    }
    (void)nthreads;
    return 0;
}

/* Full statistic: num = max_o num(o), den = n_P*n_Q, argmax = smallest pooled origin index attaining num
 * (reading R7). Returns 0 on success. */
int oracle_ddks(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int ties_gt, int nthreads,
                uint64_t* num, uint64_t* den, double* D, int64_t* argmax)
{
    int64_t N = n_P + n_Q;
    if (d < 1 || d > 20 || n_P < 1 || n_Q < 1) return 1;
    uint64_t* per = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
    if (!per) return 2;
    int rc = oracle_ddks_per_origin(P, n_P, Q, n_Q, d, ties_gt, 0, N, per, nthreads);
    if (rc) { free(per); return rc; }
    uint64_t best = 0;
    int64_t arg = 0;
    for (int64_t o = 0; o < N; ++o)
        if (per[o] > best) { best = per[o]; arg = o; }
    free(per);
    *num = best;
    *den = (uint64_t)n_P * (uint64_t)n_Q;
    *D = (double)(*num) / (double)(*den);
    *argmax = arg;
    return 0;
}

/* Batch: item b is the pair (P + b*n_P*d, Q + b*n_Q*d); each item is the definition above. */
int oracle_ddks_batch(const float* P, const float* Q, int64_t B, int64_t n_P, int64_t n_Q, int d, int ties_gt,
                      int nthreads, uint64_t* num_out)
{
    for (int64_t b = 0; b < B; ++b) {
        uint64_t num, den; double D; int64_t arg;
        int rc = oracle_ddks(P + b * n_P * d, n_P, Q + b * n_Q * d, n_Q, d, ties_gt, nthreads, &num, &den, &D, &arg);
        if (rc) return rc;
        num_out[b] = num;
    }
    return 0;
}

/* Permutation null: for permutation j, P' = pooled[perm_j[0..n_P)], Q' = pooled[perm_j[n_P..N)],
 * then the definition above. observed = identity split. p = (1 + #{null_j >= observed}) / (1 + n_perm),
 * returned as the exact numerator p_num (denominator 1 + n_perm) and as a double. */
int oracle_permutation_null(const float* pooled, int64_t n_P, int64_t n_Q, int d, const int32_t* perms,
                            int64_t n_perm, int ties_gt, int nthreads, uint64_t* null_num, uint64_t* observed,
                            int64_t* p_num, double* p_value)
{
    int64_t N = n_P + n_Q;
    uint64_t den; double D; int64_t arg;
    int rc = oracle_ddks(pooled, n_P, pooled + n_P * d, n_Q, d, ties_gt, nthreads, observed, &den, &D, &arg);
    if (rc) return rc;
    float* Pp = (float*)malloc(sizeof(float) * (size_t)(n_P * d));
    float* Qp = (float*)malloc(sizeof(float) * (size_t)(n_Q * d));
    int64_t ge = 0;
    for (int64_t j = 0; j < n_perm; ++j) {
        const int32_t* pj = perms + j * N;
        for (int64_t i = 0; i < n_P; ++i) memcpy(Pp + i * d, pooled + (int64_t)pj[i] * d, sizeof(float) * d);
        for (int64_t i = 0; i < n_Q; ++i) memcpy(Qp + i * d, pooled + (int64_t)pj[n_P + i] * d, sizeof(float) * d);
        rc = oracle_ddks(Pp, n_P, Qp, n_Q, d, ties_gt, nthreads, &null_num[j], &den, &D, &arg);
        if (rc) break;
        if (null_num[j] >= *observed) ge += 1;
    }
    free(Pp);
    free(Qp);
    *p_num = 1 + ge;
    *p_value = (double)(1 + ge) / (double)(1 + n_perm);
    return rc;
}

/* ===================================================================================================================
 * Analytic significance (§3). TEST INFRASTRUCTURE ONLY, like the above.
 *
 *   M_T[i,k]  = # points of T (= Q) in orthant i about test point k, test points = all pooled points
 *   lambda_ik = (M_T[i,k] + 1) / (N_T + 2)                                           (Bayes estimator)
 *   p(n:m,l)  = C(m,n) l^n (1-l)^(m-n)                                              (binomial pmf)
 *               or, with `poisson`, the Poisson pmf e^{-ml} (ml)^n / n!
 *   p(d<=D)   = sum over (n_P, n_T), 0<=n_P<=N_P, 0<=n_T<=N_T, with |n_P/N_P - n_T/N_T| <= D
 *               of p(n_P:N_P,l) p(n_T:N_T,l)                                        (R12:
 *               "<=", decided exactly as |n_P N_T - n_T N_P| <= num with D = num / (N_P N_T))
 *   S         = 1 - prod over the 2^d orthants i and the N test points k of p(d<=D)    (R13)
 * Written literally: for every cell, the full double sum; the product accumulated as a sum of logs.
 * ===================================================================================================================*/
#include <math.h>

/* log of the binomial (or Poisson) pmf of n successes in m trials at rate l (P:L244-250 / P:L278-281). */
double oracle_log_pmf(int64_t n, int64_t m, double l, int poisson)
{
    if (poisson) {
        double mu = (double)m * l;
        return -mu + (double)n * log(mu) - lgamma((double)n + 1.0);
    }
    return lgamma((double)m + 1.0) - lgamma((double)n + 1.0) - lgamma((double)(m - n) + 1.0)
         + (double)n * log(l) + (double)(m - n) * log1p(-l);
}

/* p(d <= D : N_P, N_T, l) with D = num / (N_P N_T): the double sum over the Delta-set band. */
double oracle_p_le(uint64_t num, int64_t N_P, int64_t N_T, double l, int poisson)
{
    double p = 0.0;
    for (int64_t nP = 0; nP <= N_P; ++nP) {
        for (int64_t nT = 0; nT <= N_T; ++nT) {
            int64_t diff = nP * N_T - nT * N_P;
            uint64_t a = (uint64_t)(diff < 0 ? -diff : diff);
            if (a <= num)
                p += exp(oracle_log_pmf(nP, N_P, l, poisson) + oracle_log_pmf(nT, N_T, l, poisson));
        }
    }
    return p;
}

/* S for the pair (P, Q): computes num (the statistic) and M_T by the loop method above, then the product.
 * Outputs: *S, *log_prod = sum of log p(d<=D) over all 2^d x N cells, *num_out. Returns 0 on success. */
int oracle_significance(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int ties_gt, int poisson,
                        int nthreads, double* S, double* log_prod, uint64_t* num_out)
{
    uint64_t num, den; double D; int64_t arg;
    int rc = oracle_ddks(P, n_P, Q, n_Q, d, ties_gt, nthreads, &num, &den, &D, &arg);
    if (rc) return rc;
    int64_t N = n_P + n_Q, nq = (int64_t)1 << d;
    double acc = 0.0;
#pragma omp parallel for reduction(+ : acc) schedule(dynamic, 4)
    for (int64_t k = 0; k < N; ++k) {
        const float* test = pooled_row(P, n_P, Q, d, k);
        int64_t* MT = (int64_t*)calloc((size_t)nq, sizeof(int64_t));
        for (int64_t x = 0; x < n_Q; ++x) MT[oracle_orthant_index(test, Q + x * d, d, ties_gt)] += 1;
        for (int64_t i = 0; i < nq; ++i) {
            double l = ((double)MT[i] + 1.0) / ((double)n_Q + 2.0);
            acc += log(oracle_p_le(num, n_P, n_Q, l, poisson));
        }
        free(MT);
    }
    *log_prod = acc;
    *S = 1.0 - exp(acc);
    *num_out = num;
    return 0;
}

/* ===================================================================================================================
 * Approximations of §2.2.2-2.2.3 (SURVEY.md §8f NEXT-3 vdKS, NEXT-4 rdKS). TEST INFRASTRUCTURE ONLY, like the above.
 * Both start with NormalizeData ("shifted and rescaled to be between 0 and 1"): per dimension m, over the
 * pooled points, x' = (x - min_m) / (max_m - min_m) in double; a constant dimension maps to 0.5 (R15).
 * ===================================================================================================================*/
void oracle_normalize_pair(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, double* out /* [N][d] */)
{
    int64_t N = n_P + n_Q;
    for (int m = 0; m < d; ++m) {
        double mn = (double)pooled_row(P, n_P, Q, d, 0)[m], mx = mn;
        for (int64_t i = 1; i < N; ++i) {
            double x = (double)pooled_row(P, n_P, Q, d, i)[m];
            if (x < mn) mn = x;
            if (x > mx) mx = x;
        }
        for (int64_t i = 0; i < N; ++i) {
            double x = (double)pooled_row(P, n_P, Q, d, i)[m];
            out[i * d + m] = (mx > mn) ? (x - mn) / (mx - mn) : 0.5;
        }
    }
}

/* Alg. 1 IndexFromPoint (SPEC S:L190-197 voxel_index): cell c_m = min(floor(x'_m k), k - 1), flat = sum c_m k^m. */
int64_t oracle_voxel_index(const double* xn, int d, int64_t k)
{
    int64_t flat = 0, stride = 1;
    for (int m = 0; m < d; ++m) {
        int64_t c = (int64_t)floor(xn[m] * (double)k);
        if (c > k - 1) c = k - 1;
        if (c < 0) c = 0;
        flat += c * stride;
        stride *= k;
    }
    return flat;
}

/* vdKS, Alg. 1 step by step:
 *   VoxelList[id][index] += 1 for every point (id 0 = P, 1 = T = Q), FilledVoxels = indices with a point;
 *   Diff = VoxelList[1]/n_T - VoxelList[0]/n_P, kept exact as the integer diff[v] = cQ[v] n_P - cP[v] n_Q
 *   (= n_P n_Q x Diff; R16);
 *   for every filled voxel v: SumOrthants(Diff at v) = for every voxel u, orthant bit m = [u_m >= v_m] (the voxel
 *   itself in the all->= orthant, as Eq. 3 puts the origin; R16), sums[code] += diff[u]; TmpD = max_code |sums|;
 *   D = max over filled voxels. num = max |sum|, den = n_P n_Q, D = num / den. Returns 0 on success. */
int oracle_vdks_voxels(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t k,
                       int64_t v_begin, int64_t v_end, uint64_t* num, uint64_t* den, double* D);

int oracle_vdks(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t k,
                uint64_t* num, uint64_t* den, double* D)
{
    return oracle_vdks_voxels(P, n_P, Q, n_Q, d, k, 0, -1, num, den, D);
}

/* As oracle_vdks, with the max taken over the filled voxels of flat index range [v_begin, v_end) only (v_end < 0:
 * all); used by the multi-rank tests to check the voxel-sharded combine. */
int oracle_vdks_voxels(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t k,
                       int64_t v_begin, int64_t v_end, uint64_t* num, uint64_t* den, double* D)
{
    if (d < 1 || d > 20 || n_P < 1 || n_Q < 1 || k < 1) return 1;
    int64_t N = n_P + n_Q, V = 1;
    for (int m = 0; m < d; ++m) { V *= k; if (V > ((int64_t)1 << 28)) return 2; }
    double* xn = (double*)malloc(sizeof(double) * (size_t)(N * d));
    int64_t* cP = (int64_t*)calloc((size_t)V, sizeof(int64_t));
    int64_t* cQ = (int64_t*)calloc((size_t)V, sizeof(int64_t));
    int64_t* diff = (int64_t*)calloc((size_t)V, sizeof(int64_t));
    int64_t nq = (int64_t)1 << d;
    oracle_normalize_pair(P, n_P, Q, n_Q, d, xn);
    for (int64_t i = 0; i < N; ++i) {
        int64_t v = oracle_voxel_index(xn + i * d, d, k);
        if (i < n_P) cP[v] += 1; else cQ[v] += 1;
    }
    for (int64_t v = 0; v < V; ++v) diff[v] = cQ[v] * n_P - cP[v] * n_Q;
    uint64_t best = 0;
#pragma omp parallel
    {
        int64_t* sums = (int64_t*)malloc(sizeof(int64_t) * (size_t)nq);
        int64_t* vc = (int64_t*)malloc(sizeof(int64_t) * (size_t)d);
        int64_t* uc = (int64_t*)malloc(sizeof(int64_t) * (size_t)d);
#pragma omp for schedule(dynamic, 8) reduction(max : best)
        for (int64_t v = v_begin; v < (v_end < 0 ? V : (v_end < V ? v_end : V)); ++v) {
            if (cP[v] + cQ[v] == 0) continue;  /* not a filled voxel */
            for (int64_t q = 0; q < nq; ++q) sums[q] = 0;
            int64_t r = v;
            for (int m = 0; m < d; ++m) { vc[m] = r % k; r /= k; }
            for (int64_t u = 0; u < V; ++u) {
                int64_t s = u;
                int code = 0;
                for (int m = 0; m < d; ++m) { uc[m] = s % k; s /= k; code += (uc[m] >= vc[m]) << m; }
                sums[code] += diff[u];
            }
            for (int64_t q = 0; q < nq; ++q) {
                uint64_t a = (uint64_t)(sums[q] < 0 ? -sums[q] : sums[q]);
                if (a > best) best = a;
            }
        }
        free(sums); free(vc); free(uc);
    }
    free(xn); free(cP); free(cQ); free(diff);
    *num = best;
    *den = (uint64_t)n_P * (uint64_t)n_Q;
    *D = (double)best / (double)(*den);
    return 0;
}

/* Alg. 2 GetDFromCornerLists on two ascending lists, as a two-pointer merge that evaluates
 * |numC1 len(C2) - numC2 len(C1)| only once both pointers have consumed every value <= the current one (DESIGN.md
 * R17: the printed loop compares C2[0] < C1[0] and cannot advance correctly; absolute value for symmetry).
 * Returns the integer numerator; the statistic is num / (len(C1) len(C2)). */
uint64_t oracle_merged_max_diff(const double* c1, int64_t n1, const double* c2, int64_t n2)
{
    int64_t i = 0, j = 0;
    uint64_t best = 0;
    while (i < n1 || j < n2) {
        double v;
        if (i < n1 && (j >= n2 || c1[i] <= c2[j])) v = c1[i]; else v = c2[j];
        while (i < n1 && c1[i] <= v) ++i;
        while (j < n2 && c2[j] <= v) ++j;
        int64_t t = i * n2 - j * n1;
        uint64_t a = (uint64_t)(t < 0 ? -t : t);
        if (a > best) best = a;
    }
    return best;
}

static int cmp_double(const void* a, const void* b)
{
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* rdKS, Alg. 2 step by step: C = IdentifyCorners = the origin of the normalised space and the d unit
 * axis corners ("(0,0,0), (1,0,0), (0,1,0), (0,0,1)"); for each corner c: Euclidean distances
 * sqrt(sum_m (x'_m - c_m)^2) (summed m = 0..d-1) of P's and T's points, each list sorted, then
 * GetDFromCornerLists; D = max over corners. num/den as above; *arg_corner = first corner attaining num. */
int oracle_rdks_corners(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t c_begin,
                        int64_t c_end, uint64_t* num, uint64_t* den, double* D, int64_t* arg_corner);

int oracle_rdks(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d,
                uint64_t* num, uint64_t* den, double* D, int64_t* arg_corner)
{
    return oracle_rdks_corners(P, n_P, Q, n_Q, d, 0, d + 1, num, den, D, arg_corner);
}

/* As oracle_rdks over corners [c_begin, c_end) only (multi-rank tests: corner-sharded combine); *arg_corner = -1 if
 * the range is empty. */
int oracle_rdks_corners(const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t c_begin,
                        int64_t c_end, uint64_t* num, uint64_t* den, double* D, int64_t* arg_corner)
{
    if (d < 1 || n_P < 1 || n_Q < 1) return 1;
    int64_t N = n_P + n_Q;
    double* xn = (double*)malloc(sizeof(double) * (size_t)(N * d));
    oracle_normalize_pair(P, n_P, Q, n_Q, d, xn);
    uint64_t best = 0;
    int64_t arg = c_begin < c_end ? c_begin : -1;
#pragma omp parallel
    {
        double* dP = (double*)malloc(sizeof(double) * (size_t)n_P);
        double* dQ = (double*)malloc(sizeof(double) * (size_t)n_Q);
        double* c = (double*)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
        for (int64_t ci = c_begin; ci < c_end; ++ci) {
            for (int m = 0; m < d; ++m) c[m] = (ci >= 1 && m == ci - 1) ? 1.0 : 0.0;
            for (int64_t i = 0; i < N; ++i) {
                double s = 0.0;
                for (int m = 0; m < d; ++m) { double t = xn[i * d + m] - c[m]; s += t * t; }
                if (i < n_P) dP[i] = sqrt(s); else dQ[i - n_P] = sqrt(s);
            }
            qsort(dP, (size_t)n_P, sizeof(double), cmp_double);
            qsort(dQ, (size_t)n_Q, sizeof(double), cmp_double);
            uint64_t t = oracle_merged_max_diff(dP, n_P, dQ, n_Q);
#pragma omp critical
            {
                if (t > best || (t == best && ci < arg)) { best = t; arg = ci; }
            }
        }
        free(dP); free(dQ); free(c);
    }
    free(xn);
    *num = best;
    *den = (uint64_t)n_P * (uint64_t)n_Q;
    *D = (double)best / (double)(*den);
    *arg_corner = arg;
    return 0;
}
