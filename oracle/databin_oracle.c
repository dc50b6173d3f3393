/*
 * databin_oracle.c -- the CPU oracle for the in situ DataBin hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * code.  The product library (paper_2310_02926_b200/) never links, imports
 * or executes it, and shares no code, header, table or constant generator
 * with it.
 *
 * What it computes (arXiv 2310.02926, Sec. 4.2 "In Situ Data Binning",
 * PAPER.md:469-472):
 *   "data binning specifies a subset of the variables to use as the
 *    coordinate axes of a uniform Cartesian mesh ... For each realization,
 *    the values of the coordinate variables locate the mesh cell, or bin,
 *    to which the realization belongs.  The low and high bounds of the mesh
 *    axes can be manually specified or obtained on the fly by calculating
 *    the minimum and maximum of the respective coordinate variables.
 *    Incrementing a per-mesh-cell counter creates a histogram ...
 *    The reduction operations we support are summation, minimum, maximum,
 *    and average."
 * plus the multi-rank combine of PAPER.md:479 ("parallelized with MPI").
 *
 * The method is exact (no approximation), so this file is the plain
 * definition written out: one sequential pass in ascending row index, fp64,
 * compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 * Readings of what the paper leaves open are the DESIGN.md "Readings"
 * table entries R1..R12 (mirroring SURVEY.md §8(c) Q1..Q16); each is cited
 * where it is used below.
 *
 * Pins (tests/test_oracle.py, run with -m "not gpu"): worked examples
 * WE1-WE8, library-routine special cases (numpy histogramdd / bincount /
 * ufunc.at on inputs kept away from bin edges), closed forms on dyadic
 * grids, integer-exact sums, math.fsum error bounds, invariants and
 * partition-mode laws.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_DIM 3

/* ---- IEEE totalOrder on non-NaN doubles (reading R6: -0.0 < +0.0) ---- */
/* a strictly before b in IEEE 754 totalOrder, for non-NaN a, b. */
static int total_order_less(double a, double b)
{
    if (a < b) return 1;
    if (a > b) return 0;
    /* a == b numerically: only the pair (-0.0, +0.0) is ordered. */
    return signbit(a) && !signbit(b);
}

/* ---- Automatic bounds ("obtained on the fly by
 * calculating the minimum and maximum of the respective coordinate
 * variables"; readings R3/R4) ----
 * NaN rows do not define bounds (reading R4).  Returns 0 on success, -1 when
 * an axis has no non-NaN value (n == 0 included: degenerate). */
int oracle_bounds(int ndim, int64_t n, const double *const *axes,
                  double *lo, double *hi)
{
    if (n <= 0) return -1;
    for (int d = 0; d < ndim; ++d) {
        int seen = 0;
        double mn = 0.0, mx = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double x = axes[d][i];
            if (x != x) continue;
            if (!seen) {
                mn = mx = x;
                seen = 1;
            }
            if (total_order_less(x, mn)) mn = x;
            if (total_order_less(mx, x)) mx = x;
        }
        if (!seen) return -1;
        lo[d] = mn;
        hi[d] = mx;
    }
    return 0;
}

/* Reading R4: a degenerate axis (lo == hi) is widened to [v-0.5, v+0.5].
 * Applied after the (possibly cross-rank) min/max. Returns -1 if the axis
 * is still degenerate after widening (|v| so large that 0.5 rounds away). */
int oracle_expand_degenerate(int ndim, double *lo, double *hi)
{
    for (int d = 0; d < ndim; ++d) {
        if (lo[d] == hi[d]) {
            lo[d] = lo[d] - 0.5;
            hi[d] = hi[d] + 0.5;
            if (!(lo[d] < hi[d])) return -1;
        }
    }
    return 0;
}

/* Reading R4: the mesh of an axis is usable only if lo < hi, both are finite,
 * and the width hi - lo and the scale res / (hi - lo) are finite (else the
 * index (x - lo) * scale of some in-bounds x is NaN or infinite and has no
 * bin).  Auto bounds that fail this are degenerate (-1 from oracle_databin);
 * manual ones are invalid arguments (-3).  Returns 1 when usable. */
int oracle_bounds_usable(int ndim, const int32_t *res, const double *lo, const double *hi)
{
    for (int d = 0; d < ndim; ++d) {
        if (!(lo[d] < hi[d]) || isinf(lo[d]) || isinf(hi[d])) return 0;
        double w = hi[d] - lo[d];
        if (isinf(w) || isinf((double)res[d] / w)) return 0;
    }
    return 1;
}

/* ---- Empty grid: the identity of every reduction (reading R5) ---- */
void oracle_grid_init(int64_t nbins, int nattr, uint64_t *count, double *sum,
                      double *sumabs, double *vmin, double *vmax)
{
    for (int64_t b = 0; b < nbins; ++b) count[b] = 0;
    for (int64_t j = 0; j < (int64_t)nattr * nbins; ++j) {
        sum[j] = 0.0;
        sumabs[j] = 0.0;
        vmin[j] = INFINITY;
        vmax[j] = -INFINITY;
    }
}

/* ---- The binning pass, rows in ascending index ----
 *
 * For axis d with bounds [lo_d, hi_d] and res_d cells (readings R1, R2):
 *   scale_d = (double)res_d / (hi_d - lo_d)          computed once
 *   row i is inside iff lo_d <= x <= hi_d on every axis (NaN is outside)
 *   k_d = min(floor((x - lo_d) * scale_d), res_d - 1)
 * Linear bin (reading R11, x fastest): b = k_0 + res_0*(k_1 + res_1*k_2).
 * Per bin: count += 1; per attribute a: sum += v (in row order, from +0.0),
 * min/max under IEEE totalOrder (reading R6).  sumabs accumulates |v| for
 * the tolerance of reading R8; it is not an output of the method.
 *
 * Accumulates into the given grid (does not clear it), so partition mode
 * can run it per block.  n_in / n_out are incremented. */
void oracle_accumulate(int ndim, const int32_t *res, const double *lo,
                       const double *hi, int64_t n, const double *const *axes,
                       int nattr, const double *const *attrs,
                       uint64_t *count, double *sum, double *sumabs,
                       double *vmin, double *vmax,
                       uint64_t *n_in, uint64_t *n_out)
{
    int64_t nbins = 1;
    double scale[ORACLE_MAX_DIM];
    for (int d = 0; d < ndim; ++d) {
        nbins *= res[d];
        scale[d] = (double)res[d] / (hi[d] - lo[d]);
    }
    for (int64_t i = 0; i < n; ++i) {
        int64_t k[ORACLE_MAX_DIM] = {0, 0, 0};
        int inside = 1;
        for (int d = 0; d < ndim; ++d) {
            double x = axes[d][i];
            if (!(lo[d] <= x && x <= hi[d])) { inside = 0; break; }
            double t = (x - lo[d]) * scale[d];
            int64_t kd = (int64_t)floor(t);
            if (kd > res[d] - 1) kd = res[d] - 1;
            k[d] = kd;
        }
        if (!inside) { *n_out += 1; continue; }
        int64_t b = k[0];
        if (ndim >= 2) b += (int64_t)res[0] * k[1];
        if (ndim >= 3) b += (int64_t)res[0] * res[1] * k[2];
        *n_in += 1;
        count[b] += 1;
        for (int a = 0; a < nattr; ++a) {
            double v = attrs[a][i];
            int64_t j = (int64_t)a * nbins + b;
            sum[j] = sum[j] + v;
            sumabs[j] = sumabs[j] + fabs(v);
            if (total_order_less(v, vmin[j])) vmin[j] = v;
            if (total_order_less(vmax[j], v)) vmax[j] = v;
        }
    }
}

/* ---- Cross-rank combine (SPEC merge, reading R12) ----
 * dst := dst (+) src, where src is the next rank in rank order: counts add,
 * sums fold left in rank order, min/max under totalOrder. */
void oracle_merge_into(int64_t nbins, int nattr,
                       uint64_t *count, double *sum, double *sumabs,
                       double *vmin, double *vmax,
                       const uint64_t *count_s, const double *sum_s,
                       const double *sumabs_s, const double *vmin_s,
                       const double *vmax_s)
{
    for (int64_t b = 0; b < nbins; ++b) count[b] += count_s[b];
    for (int64_t j = 0; j < (int64_t)nattr * nbins; ++j) {
        sum[j] = sum[j] + sum_s[j];
        sumabs[j] = sumabs[j] + sumabs_s[j];
        if (total_order_less(vmin_s[j], vmin[j])) vmin[j] = vmin_s[j];
        if (total_order_less(vmax[j], vmax_s[j])) vmax[j] = vmax_s[j];
    }
}

/* ---- Average ("average"; readings R5, R9, R12) ----
 * avg = sum / count with IEEE division; empty bins give quiet NaN. */
void oracle_finalize(int64_t nbins, int nattr, const uint64_t *count,
                     const double *sum, double *avg)
{
    for (int a = 0; a < nattr; ++a)
        for (int64_t b = 0; b < nbins; ++b) {
            int64_t j = (int64_t)a * nbins + b;
            avg[j] = count[b] ? sum[j] / (double)count[b] : NAN;
        }
}

/* ---- The whole operator, optionally in partition mode P ----
 * Rows are split into P contiguous index blocks [floor(rN/P), floor((r+1)N/P))
 * (the per-rank shards of PAPER.md:479); each block is binned into its own
 * grid, and the grids are folded in rank order 0..P-1 onto the empty grid.
 * P = 1 is the plain sequential loop.
 * bounds_auto: lo/hi are outputs (global min/max, then reading R4).
 * Returns 0, -1 (auto bounds on N == 0, an axis with no non-NaN value, or
 * realised bounds that are not usable -- reading R4), -2 (allocation
 * failure), -3 (bad arguments, unusable manual bounds included). */
int oracle_databin(int ndim, const int32_t *res, int bounds_auto,
                   double *lo, double *hi, int P, int64_t n,
                   const double *const *axes, int nattr,
                   const double *const *attrs,
                   uint64_t *count, double *sum, double *sumabs,
                   double *vmin, double *vmax, double *avg,
                   uint64_t *n_in, uint64_t *n_out)
{
    if (ndim < 1 || ndim > ORACLE_MAX_DIM || P < 1 || n < 0 || nattr < 0)
        return -3;
    int64_t nbins = 1;
    for (int d = 0; d < ndim; ++d) {
        if (res[d] < 1) return -3;
        nbins *= res[d];
    }
    if (bounds_auto) {
        if (oracle_bounds(ndim, n, axes, lo, hi) != 0) return -1;
        if (oracle_expand_degenerate(ndim, lo, hi) != 0) return -1;
        if (!oracle_bounds_usable(ndim, res, lo, hi)) return -1;
    }
    if (!oracle_bounds_usable(ndim, res, lo, hi)) return -3;

    *n_in = 0;
    *n_out = 0;
    oracle_grid_init(nbins, nattr, count, sum, sumabs, vmin, vmax);
    if (P == 1) {
        oracle_accumulate(ndim, res, lo, hi, n, axes, nattr, attrs, count,
                          sum, sumabs, vmin, vmax, n_in, n_out);
    } else {
        size_t fsz = (size_t)nattr * (size_t)nbins;
        uint64_t *c = malloc(sizeof(uint64_t) * (size_t)nbins);
        double *s = malloc(sizeof(double) * (fsz ? fsz : 1));
        double *sa = malloc(sizeof(double) * (fsz ? fsz : 1));
        double *mn = malloc(sizeof(double) * (fsz ? fsz : 1));
        double *mx = malloc(sizeof(double) * (fsz ? fsz : 1));
        const double *ax[ORACLE_MAX_DIM];
        const double **at = malloc(sizeof(double *) * (nattr ? nattr : 1));
        if (!c || !s || !sa || !mn || !mx || !at) {
            free(c); free(s); free(sa); free(mn); free(mx); free(at);
            return -2;
        }
        for (int r = 0; r < P; ++r) {
            int64_t b0 = (int64_t)(((__int128)r * n) / P);
            int64_t b1 = (int64_t)(((__int128)(r + 1) * n) / P);
            for (int d = 0; d < ndim; ++d) ax[d] = axes[d] + b0;
            for (int a = 0; a < nattr; ++a) at[a] = attrs[a] + b0;
            oracle_grid_init(nbins, nattr, c, s, sa, mn, mx);
            oracle_accumulate(ndim, res, lo, hi, b1 - b0, ax, nattr, at,
                              c, s, sa, mn, mx, n_in, n_out);
            oracle_merge_into(nbins, nattr, count, sum, sumabs, vmin, vmax,
                              c, s, sa, mn, mx);
        }
        free(c); free(s); free(sa); free(mn); free(mx); free(at);
    }
    oracle_finalize(nbins, nattr, count, sum, avg);
    return 0;
}

/* ---- Exact sums (reading R20) ----
 * The paper's sum reduction over a bin is, as a real number,
 * the exact sum of the bin's values; its atomic GPU evaluation
 * rounds in an unspecified order.  The exact-sum mode defines the output as
 * that exact real sum rounded ONCE to the nearest double (ties to even),
 * which no summation order changes.  Plain definition: an integer
 * accumulator in units of 2^-1074 (the spacing of every finite double) wide
 * enough for any sum of finite doubles, added to exactly, rounded once.
 * Zero sums are +0.0 (the row-order fold from +0.0 of reading R5 also gives
 * +0.0 for every zero result).  Precondition: finite values (reading R7). */
#define XL 36 /* 64-bit limbs, two's complement, bit 0 = 2^-1074 (2304 bits) */
typedef struct { uint64_t w[XL]; } oracle_xacc;

static void xacc_clear(oracle_xacc *A) { memset(A->w, 0, sizeof A->w); }

/* A += (-1)^s * m * 2^p (units of 2^-1074), m < 2^53, 0 <= p <= 2045 */
static void xacc_add(oracle_xacc *A, double v)
{
    uint64_t bits;
    memcpy(&bits, &v, 8);
    int s = (int)(bits >> 63);
    int e = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & ((1ull << 52) - 1);
    if (e == 0) e = 1; else m |= 1ull << 52;   /* subnormals share exponent 1 */
    if (m == 0) return;
    int p = e - 1;                             /* v = m * 2^(e - 1075) = m * 2^(p - 1074) */
    int L = p / 64, sh = p % 64;
    uint64_t part[3] = {m << sh, sh ? (m >> (64 - sh)) : 0, 0};
    if (!s) {
        unsigned carry = 0;
        for (int j = L; j < XL; ++j) {
            uint64_t add = j - L < 3 ? part[j - L] : 0;
            uint64_t t = A->w[j] + add;
            unsigned c1 = t < add;
            uint64_t t2 = t + carry;
            unsigned c2 = t2 < t;
            A->w[j] = t2;
            carry = c1 | c2;
            if (j - L >= 2 && !carry) break;
        }
    } else {
        unsigned borrow = 0;
        for (int j = L; j < XL; ++j) {
            uint64_t sub = j - L < 3 ? part[j - L] : 0;
            uint64_t t = A->w[j] - sub;
            unsigned b1 = A->w[j] < sub;
            uint64_t t2 = t - borrow;
            unsigned b2 = t < (uint64_t)borrow;
            A->w[j] = t2;
            borrow = b1 | b2;
            if (j - L >= 2 && !borrow) break;
        }
    }
}

static int xacc_bit(const oracle_xacc *A, int i) { return (int)((A->w[i / 64] >> (i % 64)) & 1u); }

/* The accumulator's exact value rounded once to the nearest double (ties to
 * even); beyond the largest finite double -> +-inf. */
static double xacc_round(const oracle_xacc *A0)
{
    oracle_xacc A = *A0;
    int neg = (int)(A.w[XL - 1] >> 63);
    if (neg) { /* magnitude of a two's complement value: invert and add one */
        unsigned carry = 1;
        for (int j = 0; j < XL; ++j) {
            uint64_t t = ~A.w[j] + carry;
            carry = carry && t == 0;
            A.w[j] = t;
        }
    }
    int H = -1; /* highest set bit */
    for (int i = 64 * XL - 1; i >= 0; --i)
        if (xacc_bit(&A, i)) { H = i; break; }
    if (H < 0) return 0.0;
    uint64_t out;
    if (H <= 52) {
        /* fewer than 54 significant bits above 2^-1074: exactly a subnormal, or
         * the smallest normal binade whose bit pattern is the integer itself */
        out = A.w[0] & ((1ull << 53) - 1);
    } else {
        int shift = H - 52;
        uint64_t M = 0;
        for (int i = 52; i >= 0; --i) M = (M << 1) | (uint64_t)xacc_bit(&A, shift + i);
        int round = xacc_bit(&A, shift - 1), sticky = 0;
        for (int i = shift - 2; i >= 0 && !sticky; --i) sticky = xacc_bit(&A, i);
        if (round && (sticky || (M & 1u))) M += 1;
        if (M == (1ull << 53)) { M >>= 1; shift += 1; }
        int biased = shift + 1; /* value = M * 2^(shift - 1074), M in [2^52, 2^53) */
        if (biased >= 2047) out = 0x7ff0000000000000ull;
        else out = ((uint64_t)biased << 52) | (M & ((1ull << 52) - 1));
    }
    if (neg) out |= 1ull << 63;
    double r;
    memcpy(&r, &out, 8);
    return r;
}

/* Exactly rounded sum of v[0..n). */
double oracle_exact_sum(int64_t n, const double *v)
{
    oracle_xacc A;
    xacc_clear(&A);
    for (int64_t i = 0; i < n; ++i) xacc_add(&A, v[i]);
    return xacc_round(&A);
}

/* Per-bin exactly rounded sums of every attribute (same binning pass as
 * oracle_accumulate, bounds already realised): sum[a*nbins + b].
 * Returns 0, or -2 when the accumulators cannot be allocated. */
int oracle_exact_sums(int ndim, const int32_t *res, const double *lo, const double *hi,
                      int64_t n, const double *const *axes, int nattr,
                      const double *const *attrs, double *sum)
{
    int64_t nbins = 1;
    double scale[ORACLE_MAX_DIM];
    for (int d = 0; d < ndim; ++d) {
        nbins *= res[d];
        scale[d] = (double)res[d] / (hi[d] - lo[d]);
    }
    size_t na = (size_t)nattr * (size_t)nbins;
    oracle_xacc *acc = calloc(na ? na : 1, sizeof(oracle_xacc));
    if (!acc) return -2;
    for (int64_t i = 0; i < n; ++i) {
        int64_t k[ORACLE_MAX_DIM] = {0, 0, 0};
        int inside = 1;
        for (int d = 0; d < ndim; ++d) {
            double x = axes[d][i];
            if (!(lo[d] <= x && x <= hi[d])) { inside = 0; break; }
            int64_t kd = (int64_t)floor((x - lo[d]) * scale[d]);
            if (kd > res[d] - 1) kd = res[d] - 1;
            k[d] = kd;
        }
        if (!inside) continue;
        int64_t b = k[0];
        if (ndim >= 2) b += (int64_t)res[0] * k[1];
        if (ndim >= 3) b += (int64_t)res[0] * res[1] * k[2];
        for (int a = 0; a < nattr; ++a) xacc_add(&acc[(size_t)a * nbins + b], attrs[a][i]);
    }
    for (size_t j = 0; j < na; ++j) sum[j] = xacc_round(&acc[j]);
    free(acc);
    return 0;
}

/* ---- Automatic device selection, Eq. (1) ----
 *   d = ( r mod n_u * s + d_0 ) mod n_a
 * read (reading R14) as ((r mod n_u) * s + d_0) mod n_a, which is also the
 * C precedence of the typeset expression.  Defaults n_u = n_a, s = 1,
 * d_0 = 0 are the caller's to pass. */
int oracle_eq1_device(int r, int n_u, int s, int d0, int n_a)
{
    return ((r % n_u) * s + d0) % n_a;
}
