// xsum.cuh -- exact sums (BIN_SUM_EXACT, reading R20; SURVEY.md
// 8(f) row 3): each bin's sum is its exact real sum rounded once.
//
// Every finite double is an integer multiple of 2^-1074, so the exact sum of
// any set of them is an integer in those units.  It is held per (summed
// attribute, bin) as XD signed 64-bit "digits" in carry-save form: digit k
// carries weight 2^(32k) units, receives 32-bit chunks only (|chunk| < 2^32)
// through native L2 reductions (REDG.ADD.64 of the two's-complement chunk), so
// the order of additions never matters and no carry crosses digits until the
// finalize normalises and rounds.  Layout: xs[(slot * XD + k) * B + b]
// (digit-major: the finalize reads each digit coalesced over bins).
//
// Sources of chunks: (1) a value taking a global path (rows outside a CTA's
// window, values outside the fixed-point range): v = +-m * 2^(p - 1074),
// m < 2^53 -> m << (p mod 32) split into 3 chunks at digit p / 32;
// (2) a CTA's flushed window sum: the exact 96-bit integer Q at scale 2^-F
// (values in the fixed range are exact on that grid, dev_common.cuh) ->
// |Q| << ((1074 - F) mod 32) split into 4 chunks.  Safe while a bin receives
// fewer than 2^30 chunks per digit per execute (checked at bin_execute).
//
// The digits a CTA touched are tracked in shared memory (min digit, -max
// digit, per summed attribute) and published to xrange[2 * nsum] once per
// CTA; init zeroes exactly that range of the slot's previous execute, and the
// finalize reads only it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"

namespace db {

constexpr int XD = XD_DIGITS;  // 66 digits: bits 0..2111 in units of 2^-1074 (finite doubles reach bit 2097)
constexpr int XR_EMPTY = 0x7f7f7f7f;  // reset value of both xrange words (memset byte 0x7f)

__device__ __forceinline__ void x_red(long long *p, long long c) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(c) : "memory");
}

// Shared-memory digit range of this CTA: r[2s] = min digit, r[2s+1] = -max digit.
__device__ __forceinline__ void xr_note(int *sxr, int slot, int klo, int khi) {
    int *r = sxr + 2 * slot;
    if (klo < *(volatile int *)&r[0]) atomicMin(&r[0], klo);
    if (-khi < *(volatile int *)&r[1]) atomicMin(&r[1], -khi);
}
__device__ __forceinline__ void xr_init(int *sxr) {
    if (threadIdx.x < 2 * BIN_MAX_ATTR) sxr[threadIdx.x] = XR_EMPTY;
}
// after a __syncthreads()
__device__ __forceinline__ void xr_publish(const int *sxr, int nsum, int *xrange) {
    if (threadIdx.x < 2 * nsum && sxr[threadIdx.x] != XR_EMPTY) atomicMin(&xrange[threadIdx.x], sxr[threadIdx.x]);
}

// + v (finite) into digit row (slot, b)
__device__ __forceinline__ void xsum_add_double(long long *xs, uint64_t B, int slot, uint64_t b, double v,
                                                int *sxr) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    int e = (int)((bits >> 52) & 0x7ff);
    unsigned long long m = bits & 0xfffffffffffffull;
    if (e) m |= 1ull << 52;
    else e = 1;
    if (m == 0) return;
    const int p = e - 1, k = p >> 5, sh = p & 31;
    const unsigned long long lo = m << sh;
    const long long hi = sh ? (long long)(m >> (64 - sh)) : 0ll;
    long long c0 = (long long)(lo & 0xffffffffull), c1 = (long long)(lo >> 32), c2 = hi;
    if (bits >> 63) c0 = -c0, c1 = -c1, c2 = -c2;
    long long *d = xs + ((uint64_t)slot * XD + k) * B + b;
    if (c0) x_red(d, c0);
    if (c1) x_red(d + B, c1);
    if (c2) x_red(d + 2 * B, c2);
    xr_note(sxr, slot, k, c2 ? k + 2 : k + 1);
}

// + (Q96 - cnt * off) * 2^-F, Q96 = hi:mid:lo (the window's exact fixed-point sum)
__device__ __forceinline__ void xsum_add_fixed(long long *xs, uint64_t B, int slot, uint64_t b, uint32_t lo,
                                               uint32_t mid, uint32_t hi, unsigned long long cnt, long long off,
                                               int F, int *sxr) {
    const unsigned __int128 qp = ((unsigned __int128)hi << 64) | ((unsigned __int128)mid << 32) | lo;
    const __int128 q = (__int128)qp - (__int128)cnt * (__int128)off;
    if (q == 0) return;
    const bool neg = q < 0;
    const unsigned __int128 mag = neg ? (unsigned __int128)(-q) : (unsigned __int128)q;  // < 2^96
    const int p0 = 1074 - F, k = p0 >> 5, sh = p0 & 31;
    const unsigned __int128 s = mag << sh;  // < 2^127
    long long *d = xs + ((uint64_t)slot * XD + k) * B + b;
    int top = k;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        long long c = (long long)(unsigned)(s >> (32 * j));
        if (!c) continue;
        x_red(d + (uint64_t)j * B, neg ? -c : c);
        top = k + j;
    }
    xr_note(sxr, slot, k, top);
}

// bits [s, s + 64) of the nonnegative limb vector u[0..L) whose limb 0 sits at bit `base`
__device__ __forceinline__ unsigned long long x_win64(const unsigned *u, int L, int base, int s) {
    unsigned long long r = 0;
    for (int j = 0; j < L; ++j) {
        const int a = base + 32 * j - s;  // limb j's position relative to s
        if (a >= 64 || a <= -32) continue;
        r |= a >= 0 ? ((unsigned long long)u[j] << a) : ((unsigned long long)u[j] >> (-a));
    }
    return r;
}

// any bit below absolute position s
__device__ __forceinline__ bool x_sticky(const unsigned *u, int L, int base, int s) {
    for (int j = 0; j < L; ++j) {
        const int a = base + 32 * j;
        if (a >= s) break;
        const int nb = s - a;  // bits of this limb below s
        const unsigned mask = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
        if (u[j] & mask) return true;
    }
    return false;
}

// The exact value sum_k d[k - klo] * 2^(32k) (units 2^-1074) of the digits
// [klo, khi], rounded once to the nearest double (ties to even); +-inf beyond
// DBL_MAX; zero -> +0.0.
__device__ __noinline__ static double xsum_round_digits(const long long *d, int klo, int khi) {
    if (klo > khi) return 0.0;
    unsigned u[XD + 4];
    long long carry = 0;
    int L = 0;
    for (int k = klo; k <= khi; ++k) {
        const long long t = d[k - klo] + carry;
        u[L++] = (unsigned)t;
        carry = t >> 32;  // arithmetic: the signed carry into the next digit
    }
    while (carry != 0 && carry != -1 && L < XD + 4) {
        u[L++] = (unsigned)carry;
        carry >>= 32;
    }
    const bool neg = carry == -1;
    if (neg) {  // magnitude: two's complement negate of the L-limb vector
        unsigned c = 1;
        for (int j = 0; j < L; ++j) {
            const unsigned t = ~u[j] + c;
            c = (c && t == 0) ? 1u : 0u;
            u[j] = t;
        }
    }
    int t = L - 1;
    while (t >= 0 && u[t] == 0) --t;
    if (t < 0) return 0.0;
    const int base = 32 * klo;
    const int H = base + 32 * t + (31 - __clz(u[t]));  // highest set bit (units 2^-1074)
    unsigned long long out;
    if (H <= 52) {
        out = x_win64(u, L, base, 0) & ((1ull << 53) - 1);  // the bit pattern is the integer itself
    } else {
        int shift = H - 52;
        unsigned long long M = x_win64(u, L, base, shift) & ((1ull << 53) - 1);
        const bool rnd = (x_win64(u, L, base, shift - 1) & 1ull) != 0;
        const bool sticky = x_sticky(u, L, base, shift - 1);
        if (rnd && (sticky || (M & 1ull))) ++M;
        if (M == (1ull << 53)) {
            M >>= 1;
            ++shift;
        }
        const int biased = shift + 1;
        out = biased >= 2047 ? 0x7ff0000000000000ull : (((unsigned long long)biased << 52) | (M & ((1ull << 52) - 1)));
    }
    if (neg) out |= 1ull << 63;
    return __longlong_as_double((long long)out);
}

// Digit row (slot, b) of one rank's accumulator, rounded once.
__device__ __forceinline__ double xsum_round(const long long *xs, uint64_t B, int slot, uint64_t b, int klo, int khi) {
    long long d[XD];
    for (int k = klo; k <= khi; ++k) d[k - klo] = __ldcg(xs + ((uint64_t)slot * XD + k) * B + b);
    return xsum_round_digits(d, klo, khi);
}

}  // namespace db
