// synth.cuh -- seeded, counter-based synthetic particle generator.
//
// INPUT GENERATION ONLY: holds none of the DataBin method's arithmetic.  It
// is the one module both the oracle-side tests and the GPU side use
// (SURVEY.md §8(d) input recipe).
//
// Every value is a pure function of (seed, stream, global row index), so a
// rank's shard equals the same index range of the single-GPU set, and the
// host and device builds produce identical bits: only IEEE correctly
// rounded operations are used (+ - * / sqrt), with FMA contraction disabled
// (explicit _rn intrinsics on the device, -ffp-contract=off on the host).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SYN_MUL(a, b) __dmul_rn((a), (b))
#define SYN_ADD(a, b) __dadd_rn((a), (b))
#define SYN_SUB(a, b) __dsub_rn((a), (b))
#define SYN_DIV(a, b) __ddiv_rn((a), (b))
#define SYN_SQRT(a) __dsqrt_rn((a))
#else
#include <math.h>
#define SYN_MUL(a, b) ((a) * (b))
#define SYN_ADD(a, b) ((a) + (b))
#define SYN_SUB(a, b) ((a) - (b))
#define SYN_DIV(a, b) ((a) / (b))
#define SYN_SQRT(a) sqrt((a))
#endif

// distributions
enum { SYN_UNIFORM = 0, SYN_PLUMMER = 1 };
// columns
enum { SYN_X = 0, SYN_Y = 1, SYN_Z = 2, SYN_M = 3, SYN_VX = 4, SYN_VY = 5, SYN_VZ = 6 };

// random streams (independent draws per row)
#define SYN_S_T0 0u        // Plummer radius: 3 uniforms
#define SYN_S_DIR 8u       // Plummer direction attempts: 3 per attempt
#define SYN_DIR_TRIES 32
#define SYN_S_MASS 200u
#define SYN_S_VEL 210u     // + 0..2
#define SYN_S_POS 220u     // + 0..2 (uniform positions)

#define SYN_PLUMMER_TMAX 0.9996  // t = TMAX*max(u1,u2,u3): r <= TMAX/sqrt(1-TMAX^2) ~ 35.4 a
#define SYN_CENTRAL_MASS 1000.0  // massive body at the origin

SYN_HD uint64_t syn_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

// uniform double in [0, 1) with 53 random bits
SYN_HD double syn_u01(uint64_t seed, uint32_t stream, uint64_t i) {
    uint64_t k = syn_mix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)stream * 0xD1B54A32D192ED03ULL +
                           0x632BE59BD9B4E019ULL);
    uint64_t z = syn_mix64(k + (i + 1) * 0x9E3779B97F4A7C15ULL);
    return (double)(z >> 11) * 0x1.0p-53;
}

// a + (b - a) * u, u in [0,1)
SYN_HD double syn_uniform(uint64_t seed, uint32_t stream, uint64_t i, double a, double b) {
    return SYN_ADD(a, SYN_MUL(SYN_SUB(b, a), syn_u01(seed, stream, i)));
}

// Plummer sphere with scale length 1 (positions): the 3D cumulative mass
// M(r) = (r/sqrt(1+r^2))^3, and t = max(u1,u2,u3) has CDF t^3, so
// r = t/sqrt(1-t^2) samples it exactly with IEEE ops only.  Direction:
// rejection in the cube [-1,1)^3 over a fixed number of counter-indexed
// attempts (deterministic), normalised by sqrt.
SYN_HD void syn_plummer_pos(uint64_t seed, uint64_t i, double *x, double *y, double *z) {
    double u1 = syn_u01(seed, SYN_S_T0 + 0, i), u2 = syn_u01(seed, SYN_S_T0 + 1, i),
           u3 = syn_u01(seed, SYN_S_T0 + 2, i);
    double t = u1 > u2 ? u1 : u2;
    t = t > u3 ? t : u3;
    t = SYN_MUL(SYN_PLUMMER_TMAX, t);
    double r = SYN_DIV(t, SYN_SQRT(SYN_SUB(1.0, SYN_MUL(t, t))));
    double a = 1.0, b = 0.0, c = 0.0, s = 1.0;
    for (int k = 0; k < SYN_DIR_TRIES; ++k) {
        double aa = syn_uniform(seed, SYN_S_DIR + 3 * k + 0, i, -1.0, 1.0);
        double bb = syn_uniform(seed, SYN_S_DIR + 3 * k + 1, i, -1.0, 1.0);
        double cc = syn_uniform(seed, SYN_S_DIR + 3 * k + 2, i, -1.0, 1.0);
        double ss = SYN_ADD(SYN_ADD(SYN_MUL(aa, aa), SYN_MUL(bb, bb)), SYN_MUL(cc, cc));
        if (ss > 1e-12 && ss <= 1.0) { a = aa; b = bb; c = cc; s = ss; break; }
    }
    double f = SYN_DIV(r, SYN_SQRT(s));
    *x = SYN_MUL(a, f);
    *y = SYN_MUL(b, f);
    *z = SYN_MUL(c, f);
}

// One column value of row i.
//   UNIFORM (central = 1): row 0 is the massive body at the origin at rest;
//     other rows: position U[-1,1)^3, mass U[0.5,1.5), velocity U[-1,1)^3.
//   PLUMMER: position from the Plummer sphere above, mass U[0.5,1.5),
//     velocity U[-1,1)^3 (velocities are not binned on the Plummer configs).
SYN_HD double syn_value(int dist, int central, uint64_t seed, int column, uint64_t i) {
    if (dist == SYN_UNIFORM && central && i == 0)
        return column == SYN_M ? SYN_CENTRAL_MASS : 0.0;
    switch (column) {
    case SYN_M:
        return syn_uniform(seed, SYN_S_MASS, i, 0.5, 1.5);
    case SYN_VX: case SYN_VY: case SYN_VZ:
        return syn_uniform(seed, SYN_S_VEL + (column - SYN_VX), i, -1.0, 1.0);
    default: break;
    }
    if (dist == SYN_UNIFORM) return syn_uniform(seed, SYN_S_POS + column, i, -1.0, 1.0);
    double x, y, z;
    syn_plummer_pos(seed, i, &x, &y, &z);
    return column == SYN_X ? x : (column == SYN_Y ? y : z);
}
