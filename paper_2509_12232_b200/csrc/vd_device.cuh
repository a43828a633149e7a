/*
 * vd_device.cuh -- device stages of the docking hot path (sm_100a).
 *
 * Execution model: thread-per-pose.  All poses of a CTA belong to ONE ligand,
 * so every loop below (atoms, torsions, fragment atoms, pairs) is
 * block-uniform: topology and pair parameters are read with broadcast loads
 * and control flow never diverges except at the in-box test.  Each thread
 * owns one column of a shared-memory coordinate tile
 *     S[(3*atom + axis) * B + tid]
 * so coordinate reads/writes are bank-conflict free and need no barriers.
 *
 * Stage parity (reference paths under /root/reference/pkg/src/vecdock):
 *   A1 pose   scoring/simd.py:157-222  bit-exact: __f*_rn / __d*_rn intrinsics
 *             (never contracted), fp64 where the reference uses fp64
 *   A2 inter  scoring/simd.py:89-138   box test and cell index bit-exact
 *             (IEEE division); lerps FMA'd in FAST mode
 *   A3 intra  scoring/simd.py:36-86    EXACT: the canonical sequence with fp64
 *             exp and the lane-8 fp64 summation order; FAST: rsqrt/ex2/rcp on
 *             the MUFU pipe, fp32 partial sums flushed to fp64 every 32 pairs
 */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace vd {

struct GridView {
    const float *maps;      /* (n_maps, nx, ny, nz) */
    int nx, ny, nz;
    int64_t mstride;        /* nx * ny * nz */
    float lo0, lo1, lo2, hi0, hi1, hi2, spacing;
};

struct LigView {
    int n_atoms, n_pairs, n_torsions;
    const float4 *atom;     /* centered x, y, z, charge */
    const float2 *atom2;    /* desolv factor, map index (int bits) */
    const uint32_t *pij;    /* i | j << 15 | hb << 31 */
    const float4 *pcoef;    /* a, b, qq, dsl (weight-folded) */
    const int4 *tors;       /* axis_a, axis_b, frag_lo, frag_hi */
    const int *frag;        /* ligand-local atom indices */
    float tors32, cut2, penalty;
    int elec_map, desolv_map;
};

/* energy constants (vd/energy.py:17-34, folded like vd/scoring/__init__.py:42) */
constexpr double kDielA = -8.5525;
constexpr double kDielB = 78.4 - -8.5525;
constexpr double kDielK = 7.7839;
constexpr double kLamb = 0.003627 * (78.4 - -8.5525);
constexpr double kDesolvDenom = 2.0 * 3.6 * 3.6;
constexpr float kMinR2 = 0.01f;
constexpr float kLog2e = 1.4426950408889634f;

#define VD_S(i, c) S[(3 * (i) + (c)) * B]

/* ---- A1: pose (bit-exact) ------------------------------------------------ */
template <int B>
__device__ __forceinline__ void build_pose(const LigView &L, const double *__restrict__ g,
                                           float *S)
{
    const double q0 = g[3], q1 = g[4], q2 = g[5], q3 = g[6];
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)),
                                                      __dmul_rn(q2, q2)), __dmul_rn(q3, q3)));
    const double w = __ddiv_rn(q0, nrm), x = __ddiv_rn(q1, nrm), y = __ddiv_rn(q2, nrm),
                 z = __ddiv_rn(q3, nrm);
    const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), zz = __dmul_rn(z, z);
    const double xy = __dmul_rn(x, y), xz = __dmul_rn(x, z), yz = __dmul_rn(y, z);
    const double wx = __dmul_rn(w, x), wy = __dmul_rn(w, y), wz = __dmul_rn(w, z);
    const float m00 = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(yy, zz))));
    const float m01 = __double2float_rn(__dmul_rn(2.0, __dsub_rn(xy, wz)));
    const float m02 = __double2float_rn(__dmul_rn(2.0, __dadd_rn(xz, wy)));
    const float m10 = __double2float_rn(__dmul_rn(2.0, __dadd_rn(xy, wz)));
    const float m11 = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, zz))));
    const float m12 = __double2float_rn(__dmul_rn(2.0, __dsub_rn(yz, wx)));
    const float m20 = __double2float_rn(__dmul_rn(2.0, __dsub_rn(xz, wy)));
    const float m21 = __double2float_rn(__dmul_rn(2.0, __dadd_rn(yz, wx)));
    const float m22 = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, yy))));
    const float tx = __double2float_rn(g[0]), ty = __double2float_rn(g[1]),
                tz = __double2float_rn(g[2]);
    for (int i = 0; i < L.n_atoms; ++i) {
        const float4 c = __ldg(&L.atom[i]);
        VD_S(i, 0) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(m00, c.x), __fmul_rn(m01, c.y)),
                                         __fmul_rn(m02, c.z)), tx);
        VD_S(i, 1) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(m10, c.x), __fmul_rn(m11, c.y)),
                                         __fmul_rn(m12, c.z)), ty);
        VD_S(i, 2) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(m20, c.x), __fmul_rn(m21, c.y)),
                                         __fmul_rn(m22, c.z)), tz);
    }
    for (int t = 0; t < L.n_torsions; ++t) {
        const int4 tr = __ldg(&L.tors[t]);
        const float ox = VD_S(tr.x, 0), oy = VD_S(tr.x, 1), oz = VD_S(tr.x, 2);
        const double ax = (double)__fsub_rn(VD_S(tr.y, 0), ox);
        const double ay = (double)__fsub_rn(VD_S(tr.y, 1), oy);
        const double az = (double)__fsub_rn(VD_S(tr.y, 2), oz);
        const double an = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)),
                                               __dmul_rn(az, az)));
        const float kx = __double2float_rn(__ddiv_rn(ax, an));
        const float ky = __double2float_rn(__ddiv_rn(ay, an));
        const float kz = __double2float_rn(__ddiv_rn(az, an));
        double sd, cd;
        sincos(g[7 + t], &sd, &cd);
        const float c = __double2float_rn(cd), s = __double2float_rn(sd);
        const float omc = __fsub_rn(1.0f, c);
        for (int f = tr.z; f < tr.w; ++f) {
            const int i = __ldg(&L.frag[f]);
            const float vx = __fsub_rn(VD_S(i, 0), ox), vy = __fsub_rn(VD_S(i, 1), oy),
                        vz = __fsub_rn(VD_S(i, 2), oz);
            const float dot = __fadd_rn(__fadd_rn(__fmul_rn(kx, vx), __fmul_rn(ky, vy)),
                                        __fmul_rn(kz, vz));
            const float cxx = __fsub_rn(__fmul_rn(ky, vz), __fmul_rn(kz, vy));
            const float cxy = __fsub_rn(__fmul_rn(kz, vx), __fmul_rn(kx, vz));
            const float cxz = __fsub_rn(__fmul_rn(kx, vy), __fmul_rn(ky, vx));
            const float dw = __fmul_rn(dot, omc);
            VD_S(i, 0) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(vx, c), __fmul_rn(cxx, s)),
                                             __fmul_rn(kx, dw)), ox);
            VD_S(i, 1) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(vy, c), __fmul_rn(cxy, s)),
                                             __fmul_rn(ky, dw)), oy);
            VD_S(i, 2) = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(vz, c), __fmul_rn(cxz, s)),
                                             __fmul_rn(kz, dw)), oz);
        }
    }
}

/* ---- A2: inter ------------------------------------------------------------ */
template <bool EXACT>
__device__ __forceinline__ float lerp_(float a, float b, float t)
{
    if (EXACT) return __fadd_rn(__fmul_rn(a, __fsub_rn(1.0f, t)), __fmul_rn(b, t));
    return fmaf(b, t, a * (1.0f - t));
}

template <bool EXACT>
__device__ __forceinline__ float trilerp(const float *__restrict__ m, int idx, int nz, int nyz,
                                         float fx, float fy, float fz)
{
    const float v000 = __ldg(m + idx), v001 = __ldg(m + idx + 1);
    const float v010 = __ldg(m + idx + nz), v011 = __ldg(m + idx + nz + 1);
    const float v100 = __ldg(m + idx + nyz), v101 = __ldg(m + idx + nyz + 1);
    const float v110 = __ldg(m + idx + nyz + nz), v111 = __ldg(m + idx + nyz + nz + 1);
    const float c00 = lerp_<EXACT>(v000, v100, fx), c10 = lerp_<EXACT>(v010, v110, fx);
    const float c01 = lerp_<EXACT>(v001, v101, fx), c11 = lerp_<EXACT>(v011, v111, fx);
    const float c0 = lerp_<EXACT>(c00, c10, fy), c1 = lerp_<EXACT>(c01, c11, fy);
    return lerp_<EXACT>(c0, c1, fz);
}

template <bool EXACT, int B>
__device__ __forceinline__ double inter_energy(const LigView &L, const GridView &G,
                                               const float *S)
{
    double acc = 0.0;
    const int nyz = G.ny * G.nz;
    for (int i = 0; i < L.n_atoms; ++i) {
        const float x = VD_S(i, 0), y = VD_S(i, 1), z = VD_S(i, 2);
        float term;
        if (x >= G.lo0 && x <= G.hi0 && y >= G.lo1 && y <= G.hi1 && z >= G.lo2 && z <= G.hi2) {
            const float ux = __fdiv_rn(__fsub_rn(x, G.lo0), G.spacing);
            const float uy = __fdiv_rn(__fsub_rn(y, G.lo1), G.spacing);
            const float uz = __fdiv_rn(__fsub_rn(z, G.lo2), G.spacing);
            const int ix = min((int)ux, G.nx - 2), iy = min((int)uy, G.ny - 2),
                      iz = min((int)uz, G.nz - 2);
            const float fx = __fsub_rn(ux, (float)ix), fy = __fsub_rn(uy, (float)iy),
                        fz = __fsub_rn(uz, (float)iz);
            const int idx = (ix * G.ny + iy) * G.nz + iz;
            const float4 a = __ldg(&L.atom[i]);
            const float2 a2 = __ldg(&L.atom2[i]);
            const float vt = trilerp<EXACT>(G.maps + G.mstride * __float_as_int(a2.y), idx, G.nz,
                                            nyz, fx, fy, fz);
            const float ve = trilerp<EXACT>(G.maps + G.mstride * L.elec_map, idx, G.nz, nyz, fx,
                                            fy, fz);
            const float vd = trilerp<EXACT>(G.maps + G.mstride * L.desolv_map, idx, G.nz, nyz,
                                            fx, fy, fz);
            if (EXACT)
                term = __fadd_rn(__fadd_rn(vt, __fmul_rn(a.w, ve)), __fmul_rn(a2.x, vd));
            else
                term = fmaf(a2.x, vd, fmaf(a.w, ve, vt));
        } else {
            const float dx = fmaxf(fmaxf(__fsub_rn(G.lo0, x), __fsub_rn(x, G.hi0)), 0.0f);
            const float dy = fmaxf(fmaxf(__fsub_rn(G.lo1, y), __fsub_rn(y, G.hi1)), 0.0f);
            const float dz = fmaxf(fmaxf(__fsub_rn(G.lo2, z), __fsub_rn(z, G.hi2)), 0.0f);
            const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)),
                                       __fmul_rn(dz, dz));
            term = __fmul_rn(L.penalty, __fadd_rn(__fsqrt_rn(d2), 1.0f));
        }
        acc = __dadd_rn(acc, (double)term);
    }
    return acc;
}

/* ---- A3: intra -------------------------------------------------------------- */
__device__ __forceinline__ float pair_term_exact(float dx, float dy, float dz, uint32_t w,
                                                 float4 cf, float cut2)
{
    const float r2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    if (r2 > cut2) return 0.0f;
    const float r2c = r2 > kMinR2 ? r2 : kMinR2;
    const float inv = __fdiv_rn(1.0f, r2c);
    const float i2 = __fmul_rn(inv, inv), i3 = __fmul_rn(i2, inv), i6 = __fmul_rn(i3, i3);
    const float tail = (w >> 31) ? __fmul_rn(i3, i2) : i3;
    const float well = __fsub_rn(__fmul_rn(cf.x, i6), __fmul_rn(cf.y, tail));
    const float r = __fsqrt_rn(r2c);
    const double r64 = (double)r;
    const double eps_r = __dadd_rn(kDielA, __ddiv_rn(kDielB, __dadd_rn(1.0, __dmul_rn(kDielK, exp(-__dmul_rn(kLamb, r64))))));
    const float elec = __double2float_rn(__ddiv_rn((double)cf.z, __dmul_rn(r64, eps_r)));
    const float des = __double2float_rn(__dmul_rn((double)cf.w, exp(-__ddiv_rn((double)r2, kDesolvDenom))));
    return __fadd_rn(__fadd_rn(well, elec), des);
}

__device__ __forceinline__ float pair_term_fast(float dx, float dy, float dz, uint32_t w,
                                                float4 cf, float cut2)
{
    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    const float r2c = fmaxf(r2, kMinR2);
    const float rs = rsqrtf(r2c);                 /* MUFU.RSQ */
    const float inv = rs * rs;                    /* 1 / r^2  */
    const float r = r2c * rs;                     /* r        */
    const float i2 = inv * inv, i3 = i2 * inv, i6 = i3 * i3;
    const float tail = (w >> 31) ? i3 * i2 : i3;
    const float well = fmaf(cf.x, i6, -cf.y * tail);
    /* sigmoidal dielectric: eps = A + B/(1+K e),  e = exp(-lamb r)
       elec = qq / (r eps) = qq (1 + K e) / (r (A (1 + K e) + B)) */
    const float e1 = exp2f(r * (float)(-kLamb * 1.4426950408889634));     /* MUFU.EX2 */
    const float den = fmaf((float)kDielK, e1, 1.0f);
    const float elec = __fdividef(cf.z * den, r * fmaf((float)kDielA, den, (float)kDielB));
    const float des = cf.w * exp2f(r2 * (float)(-1.4426950408889634 / kDesolvDenom)); /* MUFU.EX2 */
    const float t = (well + elec) + des;
    return r2 > cut2 ? 0.0f : t;
}

template <bool EXACT, int B>
__device__ __forceinline__ double intra_energy(const LigView &L, const float *S)
{
    const int n = L.n_pairs;
    if (EXACT) {
        /* simd lane-blocked order, lane = 8 (scoring/simd.py:58-86) */
        double lane[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int nblk = n >> 3;
        for (int blk = 0; blk < nblk; ++blk) {
#pragma unroll
            for (int l = 0; l < 8; ++l) {
                const int k = blk * 8 + l;
                const uint32_t w = __ldg(&L.pij[k]);
                const float4 cf = __ldg(&L.pcoef[k]);
                const int i = w & 0x7fff, j = (w >> 15) & 0x7fff;
                const float t = pair_term_exact(__fsub_rn(VD_S(i, 0), VD_S(j, 0)),
                                                __fsub_rn(VD_S(i, 1), VD_S(j, 1)),
                                                __fsub_rn(VD_S(i, 2), VD_S(j, 2)), w, cf, L.cut2);
                lane[l] = __dadd_rn(lane[l], (double)t);
            }
        }
        double tail = 0.0;
        for (int k = nblk * 8; k < n; ++k) {
            const uint32_t w = __ldg(&L.pij[k]);
            const float4 cf = __ldg(&L.pcoef[k]);
            const int i = w & 0x7fff, j = (w >> 15) & 0x7fff;
            tail = __dadd_rn(tail, (double)pair_term_exact(__fsub_rn(VD_S(i, 0), VD_S(j, 0)),
                                                           __fsub_rn(VD_S(i, 1), VD_S(j, 1)),
                                                           __fsub_rn(VD_S(i, 2), VD_S(j, 2)), w,
                                                           cf, L.cut2));
        }
        double tot = 0.0;
#pragma unroll
        for (int l = 0; l < 8; ++l) tot = __dadd_rn(tot, lane[l]);
        return __dadd_rn(tot, tail);
    } else {
        double acc = 0.0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k1 = min(k0 + 32, n);
            float part = 0.0f;
#pragma unroll 4
            for (int k = k0; k < k1; ++k) {
                const uint32_t w = __ldg(&L.pij[k]);
                const float4 cf = __ldg(&L.pcoef[k]);
                const int i = w & 0x7fff, j = (w >> 15) & 0x7fff;
                part += pair_term_fast(VD_S(i, 0) - VD_S(j, 0), VD_S(i, 1) - VD_S(j, 1),
                                       VD_S(i, 2) - VD_S(j, 2), w, cf, L.cut2);
            }
            acc += (double)part;
        }
        return acc;
    }
}

__device__ __forceinline__ float total32(double inter, double intra, float tors)
{
    return __fadd_rn(__fadd_rn(__double2float_rn(inter), __double2float_rn(intra)), tors);
}

}  // namespace vd
