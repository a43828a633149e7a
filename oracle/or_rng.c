/*
 * or_rng.c -- the restated GA's random stream, written for the oracle alone
 * (TEST INFRASTRUCTURE ONLY; see vd_oracle.c for who may load it).
 *
 * This file does not include or compile any product source.  It restates,
 * from the specification in DESIGN.md section 4, the counter map and the
 * three transforms the restated GA draws through, so that the device GA
 * (csrc/vd_rng.h + csrc/vd_ga.cu) is checked against an independent
 * implementation:
 *
 *   key      (global_seed, ligand_index)                     vd/ga.py:74-77 (make_rng)
 *   block    Philox4x64-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123
 *            round constants), pinned against numpy's own Philox blocks
 *            (tests/golden/philox.npz, produced by numpy)
 *   counter  (slot / 4, individual, generation, phase); word = slot % 4
 *            phase 1 init uniforms, 2 init normals (slot = quaternion
 *            component), 3 breed uniforms / integers, 4 breed normals
 *            (slot = gene index)
 *   uniform  (w >> 11) * 2^-53, numpy Generator.random's transform
 *   integer  floor(w * n / 2^64)  (multiply-high)
 *   normal   Box-Muller on words 0 and 1 of the normal's own block:
 *            sqrt(-2 ln u1) cos(2 pi u2), u1 = ((w0 >> 11) + 1) 2^-53 in (0, 1],
 *            u2 = (w1 >> 11) 2^-53; ln by the 2 atanh((m-1)/(m+1)) series
 *            (odd terms to f^25) after splitting x = m 2^e with m in
 *            [sqrt(1/2), sqrt(2)), ln 2 in fdlibm's Cody-Waite halves; cos by its
 *            Taylor series to x^24 after folding u into [0, 1/4].  Every step is
 *            an IEEE-754 correctly rounded operation (+ - * / sqrt fma), so the
 *            result is a function of the inputs alone.
 *
 * The transforms' accuracy against libm and the normals' distribution are
 * checked in tests/test_host_cpu.py; bit equality with the device stream in
 * tests/test_gpu_ga.py (>= 1e5 draws per phase).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "or_rng.h"

/* ---- Philox4x64-10 -------------------------------------------------------- */
static const uint64_t PHILOX_M[2] = {0xD2E7470EE14C6C93ULL, 0xCA5A826395121157ULL};
static const uint64_t PHILOX_W[2] = {0x9E3779B97F4A7C15ULL, 0xBB67AE8584CAA73BULL};

static inline uint64_t mul_hi(uint64_t a, uint64_t b, uint64_t *lo)
{
    const unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
    *lo = (uint64_t)p;
    return (uint64_t)(p >> 64);
}

void or_philox(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4])
{
    uint64_t x[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint64_t k[2] = {key_in[0], key_in[1]};
    for (int round = 0; round < 10; ++round) {
        if (round) {  /* key schedule: bump between rounds */
            k[0] += PHILOX_W[0];
            k[1] += PHILOX_W[1];
        }
        uint64_t lo0, lo1;
        const uint64_t hi0 = mul_hi(PHILOX_M[0], x[0], &lo0);
        const uint64_t hi1 = mul_hi(PHILOX_M[1], x[2], &lo1);
        const uint64_t y[4] = {hi1 ^ x[1] ^ k[0], lo1, hi0 ^ x[3] ^ k[1], lo0};
        memcpy(x, y, sizeof x);
    }
    memcpy(out, x, sizeof x);
}

/* ---- counter map ----------------------------------------------------------- */
uint64_t or_rng_word(const or_rng_key *key, int phase, int64_t gen, int64_t idx, int64_t slot)
{
    const uint64_t ctr[4] = {(uint64_t)slot / 4u, (uint64_t)idx, (uint64_t)gen, (uint64_t)phase};
    const uint64_t k[2] = {key->seed, key->ligand};
    uint64_t w[4];
    or_philox(ctr, k, w);
    return w[(uint64_t)slot % 4u];
}

double or_rng_uniform(uint64_t w) { return ldexp((double)(w >> 11), -53); }

uint64_t or_rng_below(uint64_t w, uint64_t n)
{
    uint64_t lo;
    return mul_hi(w, n, &lo);
}

/* ---- Box-Muller transform -------------------------------------------------- */
/* fdlibm's split of ln 2: ln2_hi has 32 trailing zero bits, so e * ln2_hi is exact */
static const double LN2_HI = 0x1.62e42feep-1;
static const double LN2_LO = 0x1.a39ef35793c76p-33;

double or_rng_ln(double x)
{
    int e;
    double m = 2.0 * frexp(x, &e);  /* x = m 2^(e-1), m in [1, 2) */
    e -= 1;
    if (m > 0x1.6a09e667f3bcdp+0) {  /* sqrt(2) rounded: fold m into [sqrt(1/2), sqrt(2)) */
        m *= 0.5;
        e += 1;
    }
    const double f = (m - 1.0) / (m + 1.0);
    const double f2 = f * f;
    /* atanh(f)/f = sum_k f^(2k) / (2k+1), Horner from the f^24 term down */
    double s = 1.0 / 25.0;
    for (int d = 23; d >= 3; d -= 2) s = fma(s, f2, 1.0 / (double)d);
    const double ln_m = 2.0 * fma(s * f2, f, f);
    const double de = (double)e;
    return fma(de, LN2_HI, ln_m) + de * LN2_LO;
}

/* 1/(2k)! for k = 12 .. 1, correctly rounded (generated from exact rationals) */
static const double INV_EVEN_FACT[12] = {
    0x1.f2cf01972f578p-80, 0x1.0ce396db7f853p-70, 0x1.e542ba4020225p-62,
    0x1.6827863b97d97p-53, 0x1.ae7f3e733b81fp-45, 0x1.93974a8c07c9dp-37,
    0x1.1eed8eff8d898p-29, 0x1.27e4fb7789f5cp-22, 0x1.a01a01a01a01ap-16,
    0x1.6c16c16c16c17p-10, 0x1.5555555555555p-5,  0x1.0000000000000p-1,
};

double or_rng_cos_2pi(double u)
{
    double v = u > 0.5 ? 1.0 - u : u;  /* cos(2 pi u) = cos(2 pi (1 - u)) */
    double sign = 1.0;
    if (v > 0.25) {                    /* cos(2 pi v) = -cos(2 pi (1/2 - v)) */
        v = 0.5 - v;
        sign = -1.0;
    }
    const double x = 0x1.921fb54442d18p+2 * v;  /* 2 pi, rounded */
    const double x2 = x * x;
    double c = INV_EVEN_FACT[0];       /* + x^24/24! */
    double sgn = -1.0;                 /* next coefficient: - x^22/22! */
    for (int k = 1; k < 12; ++k) {
        c = fma(c, x2, sgn * INV_EVEN_FACT[k]);
        sgn = -sgn;
    }
    c = fma(c, x2, 1.0);
    return sign * c;
}

double or_rng_normal(const or_rng_key *key, int phase, int64_t gen, int64_t idx, int64_t comp)
{
    const uint64_t ctr[4] = {(uint64_t)comp, (uint64_t)idx, (uint64_t)gen, (uint64_t)phase};
    const uint64_t k[2] = {key->seed, key->ligand};
    uint64_t w[4];
    or_philox(ctr, k, w);
    const double u1 = (double)((w[0] >> 11) + 1) * 0x1p-53;  /* (0, 1]: ln never sees 0 */
    const double u2 = or_rng_uniform(w[1]);
    return sqrt(-2.0 * or_rng_ln(u1)) * or_rng_cos_2pi(u2);
}

/* ---- bulk probes (tests) --------------------------------------------------- */
void or_rng_words(uint64_t seed, uint64_t ligand, int phase, int64_t gen, int64_t n_idx,
                  int64_t n_slot, uint64_t *out)
{
    const or_rng_key key = {seed, ligand};
    for (int64_t i = 0; i < n_idx; ++i)
        for (int64_t s = 0; s < n_slot; ++s)
            out[i * n_slot + s] = or_rng_word(&key, phase, gen, i, s);
}

void or_rng_normals(uint64_t seed, uint64_t ligand, int phase, int64_t gen, int64_t n_idx,
                    int64_t n_comp, double *out)
{
    const or_rng_key key = {seed, ligand};
    for (int64_t i = 0; i < n_idx; ++i)
        for (int64_t c = 0; c < n_comp; ++c)
            out[i * n_comp + c] = or_rng_normal(&key, phase, gen, i, c);
}
