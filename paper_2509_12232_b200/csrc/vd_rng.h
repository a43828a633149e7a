/*
 * vd_rng.h -- counter-based GA randomness shared by the CUDA kernels and the
 * CPU oracle (oracle/vd_ga_oracle.c), so both sides draw bit-identical
 * streams.
 *
 * Generator: Philox4x64-10 keyed (global_seed, ligand_index), the key layout
 * of vd/ga.py:74-77 (make_rng).  numpy's Generator consumes its stream
 * sequentially with data-dependent rejection (ziggurat normals), which no
 * data-parallel device code can reproduce, so the GA restated here addresses
 * every draw by counter instead:
 *
 *   counter = (c0 = slot block, c1 = individual/child, c2 = generation, c3 = phase)
 *   phase 1 init uniforms | 2 init normals | 3 breed uniforms/ints | 4 breed normals
 *
 * uniform(u64)   = (u >> 11) * 2^-53                     (numpy Generator.random)
 * integer(u64,n) = floor(u * n / 2^64)                   (multiply-high, no rejection)
 * normal         = Box-Muller on words 0,1 of its own block, with a log/cos
 *                  written here from IEEE-exact primitives only (+,-,*,/,sqrt,
 *                  explicit fma) so host and device agree to the last bit.
 */
#ifndef VD_RNG_H
#define VD_RNG_H

#include <stdint.h>

#if defined(__CUDACC__)
#define VD_HD __host__ __device__ __forceinline__
#else
#define VD_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define VD_DMUL(a, b) __dmul_rn((a), (b))
#define VD_DADD(a, b) __dadd_rn((a), (b))
#define VD_DSUB(a, b) __dsub_rn((a), (b))
#define VD_DDIV(a, b) __ddiv_rn((a), (b))
#define VD_DSQRT(a) __dsqrt_rn(a)
#define VD_DFMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <math.h>
#include <string.h>
#define VD_DMUL(a, b) ((a) * (b))
#define VD_DADD(a, b) ((a) + (b))
#define VD_DSUB(a, b) ((a) - (b))
#define VD_DDIV(a, b) ((a) / (b))
#define VD_DSQRT(a) sqrt(a)
#define VD_DFMA(a, b, c) fma((a), (b), (c))
#endif

enum { VD_PH_INIT_U = 1, VD_PH_INIT_N = 2, VD_PH_BREED_U = 3, VD_PH_BREED_N = 4 };

typedef struct { uint64_t v[4]; } vd_u64x4;

VD_HD void vd_mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo)
{
#if defined(__CUDA_ARCH__)
    *lo = a * b;
    *hi = __umul64hi(a, b);
#else
    unsigned __int128 p = (unsigned __int128)a * b;
    *lo = (uint64_t)p;
    *hi = (uint64_t)(p >> 64);
#endif
}

/* Philox4x64 with 10 rounds (Salmon et al., SC'11; Random123 constants). */
VD_HD vd_u64x4 vd_philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                uint64_t k0, uint64_t k1)
{
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0, lo0, hi1, lo1;
        vd_mulhilo64(M0, c0, &hi0, &lo0);
        vd_mulhilo64(M1, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    vd_u64x4 out = {{c0, c1, c2, c3}};
    return out;
}

VD_HD double vd_u01(uint64_t u) { return (double)(u >> 11) * (1.0 / 9007199254740992.0); }

VD_HD uint64_t vd_below(uint64_t u, uint64_t n)
{
    uint64_t hi, lo;
    vd_mulhilo64(u, n, &hi, &lo);
    return hi;
}

VD_HD int64_t vd_bits_of(double x)
{
#if defined(__CUDA_ARCH__)
    return __double_as_longlong(x);
#else
    int64_t b;
    memcpy(&b, &x, sizeof b);
    return b;
#endif
}

VD_HD double vd_double_of(int64_t b)
{
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(b);
#else
    double x;
    memcpy(&x, &b, sizeof x);
    return x;
#endif
}

/* ln(x) for normal x > 0: x = m * 2^e, m in [sqrt(1/2), sqrt(2));
 * ln m = 2 atanh(f), f = (m-1)/(m+1), |f| < 0.1716 -> odd series to f^25. */
VD_HD double vd_log(double x)
{
    int64_t b = vd_bits_of(x);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    double m = vd_double_of((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
    if (m > 1.4142135623730951) { m = VD_DMUL(m, 0.5); e += 1; }
    double f = VD_DDIV(VD_DSUB(m, 1.0), VD_DADD(m, 1.0));
    double f2 = VD_DMUL(f, f);
    double s = 1.0 / 25.0;
    s = VD_DFMA(s, f2, 1.0 / 23.0);
    s = VD_DFMA(s, f2, 1.0 / 21.0);
    s = VD_DFMA(s, f2, 1.0 / 19.0);
    s = VD_DFMA(s, f2, 1.0 / 17.0);
    s = VD_DFMA(s, f2, 1.0 / 15.0);
    s = VD_DFMA(s, f2, 1.0 / 13.0);
    s = VD_DFMA(s, f2, 1.0 / 11.0);
    s = VD_DFMA(s, f2, 1.0 / 9.0);
    s = VD_DFMA(s, f2, 1.0 / 7.0);
    s = VD_DFMA(s, f2, 1.0 / 5.0);
    s = VD_DFMA(s, f2, 1.0 / 3.0);
    double lnm = VD_DMUL(2.0, VD_DFMA(VD_DMUL(s, f2), f, f));
    const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
    double de = (double)e;
    return VD_DADD(VD_DFMA(de, LN2_HI, lnm), VD_DMUL(de, LN2_LO));
}

/* cos(2*pi*u) for u in [0, 1): fold to a in [0, 1/4] with sign, Taylor to x^24. */
VD_HD double vd_cos2pi(double u)
{
    double v = u > 0.5 ? VD_DSUB(1.0, u) : u;   /* cos even & periodic: v in [0, 1/2] */
    double sign = 1.0;
    if (v > 0.25) { v = VD_DSUB(0.5, v); sign = -1.0; }
    const double TWO_PI = 6.283185307179586;
    double x = VD_DMUL(TWO_PI, v);
    double x2 = VD_DMUL(x, x);
    /* sum_{k=0..12} (-1)^k x^(2k) / (2k)! by Horner in x2 */
    double c = 1.0 / 620448401733239439360000.0;          /* 1/24! */
    c = VD_DFMA(c, x2, -1.0 / 1124000727777607680000.0);  /* -1/22! */
    c = VD_DFMA(c, x2, 1.0 / 2432902008176640000.0);      /* 1/20! */
    c = VD_DFMA(c, x2, -1.0 / 6402373705728000.0);        /* -1/18! */
    c = VD_DFMA(c, x2, 1.0 / 20922789888000.0);           /* 1/16! */
    c = VD_DFMA(c, x2, -1.0 / 87178291200.0);             /* -1/14! */
    c = VD_DFMA(c, x2, 1.0 / 479001600.0);                /* 1/12! */
    c = VD_DFMA(c, x2, -1.0 / 3628800.0);                 /* -1/10! */
    c = VD_DFMA(c, x2, 1.0 / 40320.0);                    /* 1/8! */
    c = VD_DFMA(c, x2, -1.0 / 720.0);                     /* -1/6! */
    c = VD_DFMA(c, x2, 1.0 / 24.0);
    c = VD_DFMA(c, x2, -0.5);
    c = VD_DFMA(c, x2, 1.0);
    return VD_DMUL(sign, c);
}

/* Standard normal from one Philox block (Box-Muller on words 0 and 1). */
VD_HD double vd_normal(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                       uint64_t k1)
{
    vd_u64x4 w = vd_philox4x64_10(c0, c1, c2, c3, k0, k1);
    double u1 = VD_DMUL((double)((w.v[0] >> 11) + 1), 1.0 / 9007199254740992.0); /* (0, 1] */
    double u2 = vd_u01(w.v[1]);
    double rad = VD_DSQRT(VD_DMUL(-2.0, vd_log(u1)));
    return VD_DMUL(rad, vd_cos2pi(u2));
}

/* Word `slot` of the uniform/integer stream at (phase, gen, idx). */
VD_HD uint64_t vd_word(uint64_t slot, uint64_t idx, uint64_t gen, uint64_t phase, uint64_t k0,
                       uint64_t k1)
{
    vd_u64x4 w = vd_philox4x64_10(slot >> 2, idx, gen, phase, k0, k1);
    return w.v[slot & 3];
}

/* The same words as vd_word for one (idx, gen, phase), read at non-decreasing
 * slots: each Philox block (4 slots) is generated once instead of per word. */
typedef struct {
    uint64_t idx, gen, phase, k0, k1, blk;
    vd_u64x4 w;
} vd_words;

VD_HD vd_words vd_words_at(uint64_t idx, uint64_t gen, uint64_t phase, uint64_t k0, uint64_t k1)
{
    vd_words s;
    s.idx = idx; s.gen = gen; s.phase = phase; s.k0 = k0; s.k1 = k1;
    s.blk = ~(uint64_t)0;
    s.w.v[0] = s.w.v[1] = s.w.v[2] = s.w.v[3] = 0;
    return s;
}

VD_HD uint64_t vd_words_get(vd_words *s, uint64_t slot)
{
    if ((slot >> 2) != s->blk) {
        s->blk = slot >> 2;
        s->w = vd_philox4x64_10(s->blk, s->idx, s->gen, s->phase, s->k0, s->k1);
    }
    return s->w.v[slot & 3];
}

#endif /* VD_RNG_H */
