/*
 * vd_device.cuh -- device stages of the docking hot path (sm_100a).
 *
 * Execution model.  A CTA scores poses of ONE ligand.  Each thread owns a
 * PAIR of poses (two genotypes) whose coordinates live side by side as float2
 * in a shared-memory tile  S[(3*atom + axis) * NPP + pp],  so that the f32
 * pair arithmetic runs as packed f32x2 instructions (FFMA2/FMUL2/FADD2 on
 * sm_100a) and every broadcast load of topology or pair parameters
 * is amortised over two poses.  For large ligands TPP > 1 threads share a
 * pose pair ("sub" lanes split atoms and pairs; barriers order the torsion
 * chain), which keeps enough warps resident when 12*N bytes per pose limit
 * how many poses fit in shared memory.  All loops are CTA-uniform: topology
 * and pair parameters are broadcast reads.  Pair parameters live in shared
 * memory: the whole list, staged once per ligand, when it fits (the common
 * case, <= kResidentPairs), else streamed in tiles of kTile pairs.
 *
 * Stage parity (reference paths under /root/reference/pkg/src/vecdock):
 *   A1 pose   scoring/simd.py:157-222   bit-exact in both modes: scalar IEEE
 *             round-to-nearest intrinsics (__f*_rn, __d*_rn),
 *             never contracted; fp64 where the reference uses fp64
 *   A2 inter  scoring/simd.py:89-138    bit-exact arithmetic in both modes (IEEE
 *             division for the cell index, unfused lerps); FAST: branch-free
 *   A3 intra  scoring/simd.py:36-86     EXACT: canonical sequence, fp64 exp,
 *             lane-8 fp64 summation order; FAST: MUFU rsqrt/ex2/rcp + an FMA-pipe
 *             exp2 polynomial, f32x2
 *             math over an hb-partitioned pair stream, fp32 partials per
             kTile chunk -> fp64
 */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace vd {

/* ---- checked build (libvdb200_checked.so, -DVD_CHECKED) ------------------------------
 * compute-sanitizer is closed on this pool, so the library carries its own checks:
 *   VD_CHK(cond, site)  bounds / invariant checks; a failure sets bit `site` of a
 *                       per-translation-unit device flag word (no trap: the run goes on
 *                       and the host reads the flags, vd_debug_check_flags)
 *   vd_poison_smem()    every kernel fills its dynamic shared memory with 0xFF bytes
 *                       (NaN floats / -1 ints) before staging, so a read of a shared word
 *                       no stage wrote shows up as a NaN result
 *   VD_JITTER(k)        each warp sleeps a hashed 0-2 us at phase boundaries, so two
 *                       warps that race on shared memory without a barrier between them
 *                       see a different interleaving than in the production build; the
 *                       results must stay bit-identical (tests/test_gpu_checked.py)
 * In the production build all three compile to nothing. */
enum {
    VD_SITE_MAP = 0,     /* grid map index in [0, n_maps) */
    VD_SITE_ATOM = 1,    /* atom index (torsion axis, fragment member, pair end) < n_atoms */
    VD_SITE_FRAG = 2,    /* fragment slot inside the staged fragment list */
    VD_SITE_SMEM = 3,    /* the launch's dynamic shared memory covers the layout */
    VD_SITE_CELL = 4,    /* gather cell inside the grid */
    VD_SITE_POP = 5,     /* GA individual index < pop */
    VD_SITE_TILE = 6,    /* pair index inside the shared pair tile */
};
#ifdef VD_CHECKED
static __device__ unsigned int g_vd_chk_flags;
#define VD_CHK(cond, site)                                                        \
    do {                                                                          \
        if (!(cond)) atomicOr(&::vd::g_vd_chk_flags, 1u << (site));               \
    } while (0)
__device__ __forceinline__ unsigned dyn_smem_bytes()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void vd_poison_smem(unsigned char *smem, unsigned bytes)
{
    VD_CHK(bytes <= dyn_smem_bytes(), VD_SITE_SMEM);
    const unsigned n = dyn_smem_bytes() / 4u;
    for (unsigned k = threadIdx.x; k < n; k += blockDim.x) reinterpret_cast<unsigned *>(smem)[k] = 0xffffffffu;
    __syncthreads();
}
__device__ __forceinline__ void vd_jitter(unsigned k)
{
    unsigned h = (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^ (k * 0xC2B2AE35u);
    h ^= h >> 13;
    h *= 0x27D4EB2Fu;
    h ^= h >> 16;
    __nanosleep(h & 2047u);
}
#define VD_JITTER(k) ::vd::vd_jitter(k)
#define VD_POISON(smem, bytes) ::vd::vd_poison_smem((smem), (bytes))
#else
#define VD_CHK(cond, site) ((void)0)
#define VD_JITTER(k) ((void)0)
#define VD_POISON(smem, bytes) ((void)0)
#endif

constexpr int kTile = 256;            /* pairs per streamed tile / fp32 partial (multiple of 8) */
constexpr int kResidentPairs = 2048;  /* pair lists up to this stay resident in shared memory */

struct GridView {
    const float *maps;      /* (n_maps, nx, ny, nz) */
    int n_maps;
    int nx, ny, nz;
    int64_t mstride;        /* nx * ny * nz */
    float lo0, lo1, lo2, hi0, hi1, hi2, spacing;
    /* packed gather layout (null when the packed copy would not stay L2-resident):
     *   yz[m][node]  = the yz-brick (v[y,z], v[y,z+1], v[y+1,z], v[y+1,z+1]), 16 B, when
     *                  the touched copy fits the L2 share (zpair = 0), else "zy" z-pairs
     *                  (v[z], v[z+1]), 8 B (zpair = 1), with rows y and y+1 (y even)
     *                  interleaved: element ((x*nyp + y/2)*nz + z)*2 + (y&1)
     *   ed[2*node]   = elec yz-brick, ed[2*node+1] = desolv yz-brick (32 B, one LDG.256)
     * -> 2 LDG.128 (or 4 LDG.64) + 2 LDG.256 per atom instead of 24 scalar gathers:
     *    each scattered warp-wide load costs ~one L1TEX wavefront per lane, so the
     *    gather cost scales with load instructions, not bytes */
    const float4 *yz;
    const float4 *ed;
    int zpair;
    int nyp;                /* (ny + 1) / 2: y row pairs of a zy map */
    int64_t tstride;        /* elements per packed type map (float4 bricks or float2 zy) */
    float one;              /* 1.0f, opaque to ptxas: fma(p, one, q) is an uncontractible p + q */
};

struct LigView {
    int n_atoms, n_pairs, n_torsions, n_frag;
    const float4 *atom;     /* centered x, y, z, charge */
    const float2 *atom2;    /* desolv factor, map index (int bits) */
    const int4 *tors;       /* axis_a, axis_b, frag_lo, frag_hi */
    const int *frag;        /* ligand-local atom indices */
    /* reference order (EXACT): */
    const uint32_t *pij;    /* i | j << 15 | hb << 31 */
    const float4 *pcoef;    /* a, b, qq, dsl (weight-folded) */
    /* fast order (FAST): 12-6 pairs, then the n_pairs - n_nohb 12-10 pairs */
    const float4 *fcoef;
    const int2 *fij;        /* 3*i, 3*j: pose-tile offsets in units of NPP elements (PairTile::off) */
    int n_nohb;
    float tors32, cut2, penalty;
    int elec_map, desolv_map;
};

/* Copy a ligand's topology into shared memory (all CTA threads; caller syncs).
 * Returns a view whose topology pointers address shared memory. */
__device__ __forceinline__ LigView stage_topology(const LigView &L, unsigned char *smem,
                                                  unsigned off_atom, unsigned off_atom2,
                                                  unsigned off_tors, unsigned off_frag)
{
    LigView V = L;
    float4 *a = reinterpret_cast<float4 *>(smem + off_atom);
    float2 *a2 = reinterpret_cast<float2 *>(smem + off_atom2);
    int4 *t = reinterpret_cast<int4 *>(smem + off_tors);
    int *f = reinterpret_cast<int *>(smem + off_frag);
    const int nf = L.n_torsions ? __ldg(&L.tors[L.n_torsions - 1]).w - __ldg(&L.tors[0]).z : 0;
    const int f0 = L.n_torsions ? __ldg(&L.tors[0]).z : 0;
    for (int i = threadIdx.x; i < L.n_atoms; i += blockDim.x) {
        a[i] = __ldg(&L.atom[i]);
        a2[i] = __ldg(&L.atom2[i]);
    }
    for (int i = threadIdx.x; i < L.n_torsions; i += blockDim.x) {
        int4 r = __ldg(&L.tors[i]);
        r.z -= f0;
        r.w -= f0;
        VD_CHK(r.x >= 0 && r.x < L.n_atoms && r.y >= 0 && r.y < L.n_atoms, VD_SITE_ATOM);
        VD_CHK(r.z >= 0 && r.z <= r.w && r.w <= nf, VD_SITE_FRAG);
        t[i] = r;
    }
    for (int i = threadIdx.x; i < nf; i += blockDim.x) {
        f[i] = __ldg(&L.frag[f0 + i]);
        VD_CHK(f[i] >= 0 && f[i] < L.n_atoms, VD_SITE_ATOM);
    }
    VD_CHK(L.n_torsions == 0 || nf == L.n_frag, VD_SITE_FRAG);
    V.atom = a;
    V.atom2 = a2;
    V.tors = t;
    V.frag = f;
    return V;
}

/* energy constants (vd/energy.py:17-34, folded like vd/scoring/__init__.py:42) */
constexpr double kDielA = -8.5525;
constexpr double kDielB = 78.4 - -8.5525;
constexpr double kDielK = 7.7839;
constexpr double kLamb = 0.003627 * (78.4 - -8.5525);
constexpr double kDesolvDenom = 2.0 * 3.6 * 3.6;
constexpr float kMinR2 = 0.01f;

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
/* Exact ops for the bit-exact pose stage, applied per component with scalar
 * IEEE intrinsics.  Packed f32x2 is NOT usable naively: ptxas 12.9 fuses packed
 * multiply + add into FFMA2 (from __fmul2_rn/__fadd2_rn, from explicit
 * mul.rn/add.rn.f32x2 PTX, even under --fmad=false), which would break parity
 * with the reference's unfused float32 sequence.  The packed variant below
 * (xadd2/xsub2) writes every sum as fma(x, one, y) with a RUN-TIME one (a kernel
 * argument): ptxas cannot fold a product into it, so it is bit-exact, and it
 * halves the pose stage's FP32 instructions.  A compile-time 1.0f would be
 * contracted again (caught by the fixture tests). */
__device__ __forceinline__ float2 mul2(float2 a, float2 b)
{
    return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}
__device__ __forceinline__ float2 add2(float2 a, float2 b)
{
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b)
{
    return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
}
/* Exact packed ops (VD_POSE_PACKED): FMUL2 rounds each product; sums are written as
 * fma(a, one, b) / fma(b, -one, a) with a run-time one, which ptxas cannot contract. */
#ifndef VD_FRAG_UNROLL
#define VD_FRAG_UNROLL 2   /* fragment loop: 2 vs 4 vs 8: 1.411 / 1.419 / 1.418 ms (cfg1) */
#endif
constexpr int kFragUnroll = VD_FRAG_UNROLL;
#ifndef VD_POSE_PACKED
#define VD_POSE_PACKED 1   /* pose stage alone 0.441 -> 0.404 ms per 1M cfg1 poses; whole
                              kernel 1.557 -> 1.543 ms; cfg2 screen +1.4% */
#endif
__device__ __forceinline__ float2 xmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 xadd2(float2 a, float2 b, float2 one) { return __ffma2_rn(a, one, b); }
__device__ __forceinline__ float2 xsub2(float2 a, float2 b, float2 neg) { return __ffma2_rn(b, neg, a); }
/* Contractible packed ops for the FAST energy stage. */
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__device__ __forceinline__ float mufu_rsq(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float mufu_ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float mufu_rcp(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

/* cp.async (LDGSTS): global -> shared without staging registers */
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
#ifdef VD_CPASYNC_CA
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#define VD_S2(i, c) S[(3 * (i) + (c)) * NPP]

/* ---- A1: pose (bit-exact) ------------------------------------------------ */
__device__ __forceinline__ void rigid_of(const double *__restrict__ g, float *m, float *t)
{
    const double q0 = g[3], q1 = g[4], q2 = g[5], q3 = g[6];
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)),
                                                      __dmul_rn(q2, q2)), __dmul_rn(q3, q3)));
    const double w = __ddiv_rn(q0, nrm), x = __ddiv_rn(q1, nrm), y = __ddiv_rn(q2, nrm),
                 z = __ddiv_rn(q3, nrm);
    const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), zz = __dmul_rn(z, z);
    const double xy = __dmul_rn(x, y), xz = __dmul_rn(x, z), yz = __dmul_rn(y, z);
    const double wx = __dmul_rn(w, x), wy = __dmul_rn(w, y), wz = __dmul_rn(w, z);
    m[0] = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(yy, zz))));
    m[1] = __double2float_rn(__dmul_rn(2.0, __dsub_rn(xy, wz)));
    m[2] = __double2float_rn(__dmul_rn(2.0, __dadd_rn(xz, wy)));
    m[3] = __double2float_rn(__dmul_rn(2.0, __dadd_rn(xy, wz)));
    m[4] = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, zz))));
    m[5] = __double2float_rn(__dmul_rn(2.0, __dsub_rn(yz, wx)));
    m[6] = __double2float_rn(__dmul_rn(2.0, __dsub_rn(xz, wy)));
    m[7] = __double2float_rn(__dmul_rn(2.0, __dadd_rn(yz, wx)));
    m[8] = __double2float_rn(__dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, yy))));
    t[0] = __double2float_rn(g[0]);
    t[1] = __double2float_rn(g[1]);
    t[2] = __double2float_rn(g[2]);
}

__device__ __forceinline__ void torsion_axis(float2 ax, float2 ay, float2 az, float2 &kx,
                                             float2 &ky, float2 &kz)
{
    float k[2][3];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const double x = (double)(p ? ax.y : ax.x), y = (double)(p ? ay.y : ay.x),
                     z = (double)(p ? az.y : az.x);
        const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
        k[p][0] = __double2float_rn(__ddiv_rn(x, n));
        k[p][1] = __double2float_rn(__ddiv_rn(y, n));
        k[p][2] = __double2float_rn(__ddiv_rn(z, n));
    }
    kx = f2(k[0][0], k[1][0]);
    ky = f2(k[0][1], k[1][1]);
    kz = f2(k[0][2], k[1][2]);
}

/* Scratch floats per pose pair (TPP > 1): rigid m/t of both poses (24), the current
 * torsion's axis k of both poses (6, padded to 8), then cos/sin of every torsion of both
 * poses (4 per torsion). */
constexpr int kPoseScratch = 32;
__host__ __device__ inline int pose_scratch_floats(int n_tors) { return kPoseScratch + 4 * n_tors; }

/* Build poses g0 -> .x and g1 -> .y of the tile column S (S already offset by pp).
 * TPP > 1: the per-pose fp64 scalars are computed once and shared through the
 * scratch column X: sub 0/1 build pose 0/1's matrix and torsion axes (the chain), and
 * the cos/sin of every torsion angle -- which do not depend on the chain -- are spread
 * over all subs up front.  CTA barriers order the chain (keeping the TPP subs of a pose
 * pair in one warp with __syncwarp measured slower: the axis work then runs on half-empty
 * warps, and the bank-conflict padding it needs cost the GA an occupancy step).  The
 * caller syncs after the call (TPP > 1); the tile must be free when it is called. */
template <int NPP, int TPP>
__device__ __forceinline__ void build_pose2(const LigView &L, const double *__restrict__ g0,
                                            const double *__restrict__ g1, float2 *S, int sub,
                                            float *X, float one)
{
#if VD_POSE_PACKED
    const float2 ONE = f2(one), NEG = f2(-one);
#endif
#define VD_X(k) X[(k) * NPP]
    VD_JITTER(1);
    float2 M00, M01, M02, M10, M11, M12, M20, M21, M22, TX, TY, TZ;
    if (TPP == 1) {
        float m0[9], t0[3], m1[9], t1[3];
        rigid_of(g0, m0, t0);
        rigid_of(g1, m1, t1);
        M00 = f2(m0[0], m1[0]); M01 = f2(m0[1], m1[1]); M02 = f2(m0[2], m1[2]);
        M10 = f2(m0[3], m1[3]); M11 = f2(m0[4], m1[4]); M12 = f2(m0[5], m1[5]);
        M20 = f2(m0[6], m1[6]); M21 = f2(m0[7], m1[7]); M22 = f2(m0[8], m1[8]);
        TX = f2(t0[0], t1[0]); TY = f2(t0[1], t1[1]); TZ = f2(t0[2], t1[2]);
    } else {
        if (sub < 2) {
            float m[9], t[3];
            rigid_of(sub ? g1 : g0, m, t);
#pragma unroll
            for (int k = 0; k < 9; ++k) VD_X(12 * sub + k) = m[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) VD_X(12 * sub + 9 + k) = t[k];
        }
        /* cos/sin of every torsion angle, spread over all subs (they do not depend on
           the chain): task k = (torsion k >> 1, pose k & 1) */
        for (int k = sub; k < 2 * L.n_torsions; k += TPP) {
            double sd, cd;
            sincos(((k & 1) ? g1 : g0)[7 + (k >> 1)], &sd, &cd);
            VD_X(kPoseScratch + 4 * (k >> 1) + (k & 1)) = __double2float_rn(cd);
            VD_X(kPoseScratch + 4 * (k >> 1) + 2 + (k & 1)) = __double2float_rn(sd);
        }
        __syncthreads();
        M00 = f2(VD_X(0), VD_X(12)); M01 = f2(VD_X(1), VD_X(13)); M02 = f2(VD_X(2), VD_X(14));
        M10 = f2(VD_X(3), VD_X(15)); M11 = f2(VD_X(4), VD_X(16)); M12 = f2(VD_X(5), VD_X(17));
        M20 = f2(VD_X(6), VD_X(18)); M21 = f2(VD_X(7), VD_X(19)); M22 = f2(VD_X(8), VD_X(20));
        TX = f2(VD_X(9), VD_X(21)); TY = f2(VD_X(10), VD_X(22)); TZ = f2(VD_X(11), VD_X(23));
    }
    for (int i = sub; i < L.n_atoms; i += TPP) {
        const float4 c = L.atom[i];
        const float2 cx = f2(c.x), cy = f2(c.y), cz = f2(c.z);
#if VD_POSE_PACKED
        VD_S2(i, 0) = xadd2(xadd2(xadd2(xmul2(M00, cx), xmul2(M01, cy), ONE), xmul2(M02, cz), ONE), TX, ONE);
        VD_S2(i, 1) = xadd2(xadd2(xadd2(xmul2(M10, cx), xmul2(M11, cy), ONE), xmul2(M12, cz), ONE), TY, ONE);
        VD_S2(i, 2) = xadd2(xadd2(xadd2(xmul2(M20, cx), xmul2(M21, cy), ONE), xmul2(M22, cz), ONE), TZ, ONE);
#else
        VD_S2(i, 0) = add2(add2(add2(mul2(M00, cx), mul2(M01, cy)), mul2(M02, cz)), TX);
        VD_S2(i, 1) = add2(add2(add2(mul2(M10, cx), mul2(M11, cy)), mul2(M12, cz)), TY);
        VD_S2(i, 2) = add2(add2(add2(mul2(M20, cx), mul2(M21, cy)), mul2(M22, cz)), TZ);
#endif
    }
    if (TPP > 1) __syncthreads();
    for (int t = 0; t < L.n_torsions; ++t) {
        const int4 tr = L.tors[t];
        VD_JITTER(2 + t);
        float2 KX, KY, KZ, C, SN;
        if (TPP == 1) {
            const float2 ox = VD_S2(tr.x, 0), oy = VD_S2(tr.x, 1), oz = VD_S2(tr.x, 2);
            torsion_axis(sub2(VD_S2(tr.y, 0), ox), sub2(VD_S2(tr.y, 1), oy),
                         sub2(VD_S2(tr.y, 2), oz), KX, KY, KZ);
            double s0, c0, s1, c1;
            sincos(g0[7 + t], &s0, &c0);
            sincos(g1[7 + t], &s1, &c1);
            C = f2(__double2float_rn(c0), __double2float_rn(c1));
            SN = f2(__double2float_rn(s0), __double2float_rn(s1));
        } else {
            if (sub < 2) {
                const float ax = __fsub_rn(sub ? VD_S2(tr.y, 0).y : VD_S2(tr.y, 0).x, sub ? VD_S2(tr.x, 0).y : VD_S2(tr.x, 0).x);
                const float ay = __fsub_rn(sub ? VD_S2(tr.y, 1).y : VD_S2(tr.y, 1).x, sub ? VD_S2(tr.x, 1).y : VD_S2(tr.x, 1).x);
                const float az = __fsub_rn(sub ? VD_S2(tr.y, 2).y : VD_S2(tr.y, 2).x, sub ? VD_S2(tr.x, 2).y : VD_S2(tr.x, 2).x);
                const double x = (double)ax, y = (double)ay, z = (double)az;
                const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
                VD_X(24 + 3 * sub + 0) = __double2float_rn(__ddiv_rn(x, n));
                VD_X(24 + 3 * sub + 1) = __double2float_rn(__ddiv_rn(y, n));
                VD_X(24 + 3 * sub + 2) = __double2float_rn(__ddiv_rn(z, n));
            }
            __syncthreads();
            KX = f2(VD_X(24), VD_X(27));
            KY = f2(VD_X(25), VD_X(28));
            KZ = f2(VD_X(26), VD_X(29));
            C = f2(VD_X(kPoseScratch + 4 * t + 0), VD_X(kPoseScratch + 4 * t + 1));
            SN = f2(VD_X(kPoseScratch + 4 * t + 2), VD_X(kPoseScratch + 4 * t + 3));
        }
        const float2 ox = VD_S2(tr.x, 0), oy = VD_S2(tr.x, 1), oz = VD_S2(tr.x, 2);
        const float2 OMC = sub2(f2(1.0f), C);
#pragma unroll kFragUnroll
        for (int f = tr.z + sub; f < tr.w; f += TPP) {
            const int i = L.frag[f];
#if VD_POSE_PACKED
            const float2 vx = xsub2(VD_S2(i, 0), ox, NEG), vy = xsub2(VD_S2(i, 1), oy, NEG),
                         vz = xsub2(VD_S2(i, 2), oz, NEG);
            const float2 dot = xadd2(xadd2(xmul2(KX, vx), xmul2(KY, vy), ONE), xmul2(KZ, vz), ONE);
            const float2 cxx = xsub2(xmul2(KY, vz), xmul2(KZ, vy), NEG);
            const float2 cxy = xsub2(xmul2(KZ, vx), xmul2(KX, vz), NEG);
            const float2 cxz = xsub2(xmul2(KX, vy), xmul2(KY, vx), NEG);
            const float2 dw = xmul2(dot, OMC);
            VD_S2(i, 0) = xadd2(xadd2(xadd2(xmul2(vx, C), xmul2(cxx, SN), ONE), xmul2(KX, dw), ONE), ox, ONE);
            VD_S2(i, 1) = xadd2(xadd2(xadd2(xmul2(vy, C), xmul2(cxy, SN), ONE), xmul2(KY, dw), ONE), oy, ONE);
            VD_S2(i, 2) = xadd2(xadd2(xadd2(xmul2(vz, C), xmul2(cxz, SN), ONE), xmul2(KZ, dw), ONE), oz, ONE);
#else
            const float2 vx = sub2(VD_S2(i, 0), ox), vy = sub2(VD_S2(i, 1), oy),
                         vz = sub2(VD_S2(i, 2), oz);
            const float2 dot = add2(add2(mul2(KX, vx), mul2(KY, vy)), mul2(KZ, vz));
            const float2 cxx = sub2(mul2(KY, vz), mul2(KZ, vy));
            const float2 cxy = sub2(mul2(KZ, vx), mul2(KX, vz));
            const float2 cxz = sub2(mul2(KX, vy), mul2(KY, vx));
            const float2 dw = mul2(dot, OMC);
            VD_S2(i, 0) = add2(add2(add2(mul2(vx, C), mul2(cxx, SN)), mul2(KX, dw)), ox);
            VD_S2(i, 1) = add2(add2(add2(mul2(vy, C), mul2(cxy, SN)), mul2(KY, dw)), oy);
            VD_S2(i, 2) = add2(add2(add2(mul2(vz, C), mul2(cxz, SN)), mul2(KZ, dw)), oz);
#endif
        }
        if (TPP > 1) __syncthreads();
    }
#undef VD_X
}

/* ---- A2: inter ------------------------------------------------------------ */
/* lerp(a, b, t) = a*(1-t) + b*t with the reference's rounding in BOTH modes:
 * map corners reach ~1e12-5e17 next to receptor atoms, so any other lerp
 * formulation (e.g. fma(t, b-a, a)) moves the interpolated value by more than
 * the 1e-4 tolerance whenever the result is far smaller than its corners. */
template <bool EXACT>
__device__ __forceinline__ float lerp_(float a, float b, float t)
{
    return __fadd_rn(__fmul_rn(a, __fsub_rn(1.0f, t)), __fmul_rn(b, t));
}

#ifndef VD_PLAIN_ZPAIR
#define VD_PLAIN_ZPAIR 1
#endif
#ifndef VD_PLAIN_UNROLL
#define VD_PLAIN_UNROLL 1
#endif
constexpr int kPlainUnroll = VD_PLAIN_UNROLL;
/* (v[z], v[z+1]) of the plain layout: one LDG.64 when the pair is 8-B aligned, else two
 * LDG.32 (predicated per lane) -- 1.5 requests per corner pair instead of 2 */
template <bool ZP>
__device__ __forceinline__ float2 ld_zpair(const float *p)
{
    float2 v;
#if VD_PLAIN_ZPAIR
    if (ZP) {
    asm("{\n\t.reg .pred q;\n\t"
        "setp.eq.b32 q, %3, 0;\n\t"
        "@q ld.global.nc.v2.f32 {%0,%1}, [%2];\n\t"
        "@!q ld.global.nc.f32 %0, [%2];\n\t"
        "@!q ld.global.nc.f32 %1, [%2+4];\n\t}"
        : "=f"(v.x), "=f"(v.y)
        : "l"(p), "r"((int)(reinterpret_cast<uintptr_t>(p) & 7u)));
    return v;
    }
#endif
    v.x = __ldg(p);
    v.y = __ldg(p + 1);
    return v;
}

template <bool EXACT, bool ZP = false>
__device__ __forceinline__ float trilerp(const float *__restrict__ m, int idx, int nz, int nyz,
                                         float fx, float fy, float fz)
{
    const float2 a = ld_zpair<ZP>(m + idx), b = ld_zpair<ZP>(m + idx + nz);
    const float2 c = ld_zpair<ZP>(m + idx + nyz), d = ld_zpair<ZP>(m + idx + nyz + nz);
    const float v000 = a.x, v001 = a.y, v010 = b.x, v011 = b.y;
    const float v100 = c.x, v101 = c.y, v110 = d.x, v111 = d.y;
    const float c00 = lerp_<EXACT>(v000, v100, fx), c10 = lerp_<EXACT>(v010, v110, fx);
    const float c01 = lerp_<EXACT>(v001, v101, fx), c11 = lerp_<EXACT>(v011, v111, fx);
    const float c0 = lerp_<EXACT>(c00, c10, fy), c1 = lerp_<EXACT>(c01, c11, fy);
    return lerp_<EXACT>(c0, c1, fz);
}

/* Per-atom, per-pose gather state: cell, fractions, the corner values. */
struct Gather {
    float fx, fy, fz, pterm;
    bool inb;
    float4 t[2];   /* type-map yz corners at x and x+1 */
    float4 e[2];   /* elec yz-bricks */
    float4 d[2];   /* desolv yz-bricks */
};

__device__ __forceinline__ void cell_of(const GridView &G, float x, float y, float z, float pen,
                                        Gather &g, int &idx, int &zy)
{
    g.inb = x >= G.lo0 && x <= G.hi0 && y >= G.lo1 && y <= G.hi1 && z >= G.lo2 && z <= G.hi2;
    const float dx = fmaxf(fmaxf(__fsub_rn(G.lo0, x), __fsub_rn(x, G.hi0)), 0.0f);
    const float dy = fmaxf(fmaxf(__fsub_rn(G.lo1, y), __fsub_rn(y, G.hi1)), 0.0f);
    const float dz = fmaxf(fmaxf(__fsub_rn(G.lo2, z), __fsub_rn(z, G.hi2)), 0.0f);
    g.pterm = __fmul_rn(pen, __fadd_rn(
        __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz))), 1.0f));
    const float ux = __fdiv_rn(__fsub_rn(x, G.lo0), G.spacing);
    const float uy = __fdiv_rn(__fsub_rn(y, G.lo1), G.spacing);
    const float uz = __fdiv_rn(__fsub_rn(z, G.lo2), G.spacing);
    const int ix = min(max((int)ux, 0), G.nx - 2), iy = min(max((int)uy, 0), G.ny - 2),
              iz = min(max((int)uz, 0), G.nz - 2);
    g.fx = __fsub_rn(ux, (float)ix);
    g.fy = __fsub_rn(uy, (float)iy);
    g.fz = __fsub_rn(uz, (float)iz);
    idx = (ix * G.ny + iy) * G.nz + iz;
    zy = ((ix * G.nyp + (iy >> 1)) * G.nz + iz) * 2 + (iy & 1);
    VD_CHK(!g.inb || ((int)ux == ix && (int)uy == iy && (int)uz == iz) ||
               ux >= (float)(G.nx - 2) || uy >= (float)(G.ny - 2) || uz >= (float)(G.nz - 2),
           VD_SITE_CELL);
    VD_CHK(idx >= 0 && (int64_t)idx + (int64_t)G.ny * G.nz + G.nz + 1 < G.mstride, VD_SITE_CELL);
}

__device__ __forceinline__ void ld256(const float4 *p, float4 &lo, float4 &hi)
{
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z),
          "=f"(hi.w)
        : "l"(p));
}

/* ld256 only for lanes whose atom is in the box (on): an out-of-box lane issues no request
 * (its corners are never used: finish_packed selects the penalty term), which spares the
 * L1TEX pipe ~29% of the gathers under cfg1's sampling */
__device__ __forceinline__ void ld256_if(const float4 *p, float4 &lo, float4 &hi, bool on)
{
    asm("{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %9, 0;\n\t"
        "@q ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
        : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z),
          "=f"(hi.w)
        : "l"(p), "r"((int)on));
}

/* packed type map m (float4 units for yz-bricks; zy maps are float2 units, see GridView) */
__device__ __forceinline__ const float4 *type_map(const GridView &G, int m)
{
    return G.zpair ? reinterpret_cast<const float4 *>(reinterpret_cast<const float2 *>(G.yz) + G.tstride * m)
                   : G.yz + G.tstride * m;
}

/* The (y, y+1) z-pairs of one x-plane from a zy map: element e = zy index of (x, y, z).
 * y even: both pairs are one aligned 16-B group -> one LDG.128; y odd: they sit in two
 * groups -> two LDG.64.  Predicated loads into the same registers, so each lane costs
 * one or two L1 requests (1.5 on average, vs 2 for plain z-pairs) at the same 8 B/node. */
__device__ __forceinline__ float4 ld_zy(const float2 *tz, int e, int nz)
{
    float4 v;
    const float2 *pa = tz + e, *pb = tz + (e - (e & 1) + 2 * nz);  /* pb: row y+1 (next group) */
    asm("{\n\t.reg .pred p;\n\t"
        "setp.eq.b32 p, %6, 0;\n\t"
        "@p ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];\n\t"
        "@!p ld.global.nc.v2.f32 {%0,%1}, [%4];\n\t"
        "@!p ld.global.nc.v2.f32 {%2,%3}, [%5];\n\t}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(pa), "l"(pb), "r"(e & 1));
    return v;
}

/* ld_zy for in-box lanes only (see ld256_if) */
__device__ __forceinline__ float4 ld_zy_if(const float2 *tz, int e, int nz, bool on)
{
    float4 v;
    const float2 *pa = tz + e, *pb = tz + (e - (e & 1) + 2 * nz);
    asm("{\n\t.reg .pred p, q, r, o;\n\t"
        "setp.ne.b32 o, %7, 0;\n\t"
        "setp.eq.and.b32 p, %6, 0, o;\n\t"
        "setp.ne.and.b32 q, %6, 0, o;\n\t"
        "@p ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];\n\t"
        "@q ld.global.nc.v2.f32 {%0,%1}, [%4];\n\t"
        "@q ld.global.nc.v2.f32 {%2,%3}, [%5];\n\t}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(pa), "l"(pb), "r"(e & 1), "r"((int)on));
    return v;
}

__device__ __forceinline__ void issue_packed(const GridView &G, const float4 *__restrict__ ty,
                                             int idx, int zy, Gather &g, bool inbox_only)
{
    const int nyz = G.ny * G.nz;
    if (!inbox_only) {
        if (G.zpair) {
            /* zy z-pairs (8 B/node): half the L2 footprint of yz-bricks */
            const float2 *tz = reinterpret_cast<const float2 *>(ty);
            g.t[0] = ld_zy(tz, zy, G.nz);
            g.t[1] = ld_zy(tz, zy + 2 * G.nyp * G.nz, G.nz);
        } else {
            g.t[0] = __ldg(ty + idx);
            g.t[1] = __ldg(ty + idx + nyz);
        }
        ld256(G.ed + 2 * (int64_t)idx, g.e[0], g.d[0]);
        ld256(G.ed + 2 * (int64_t)(idx + nyz), g.e[1], g.d[1]);
        return;
    }
    const bool on = g.inb;
    if (G.zpair) {
        const float2 *tz = reinterpret_cast<const float2 *>(ty);
        g.t[0] = ld_zy_if(tz, zy, G.nz, on);
        g.t[1] = ld_zy_if(tz, zy + 2 * G.nyp * G.nz, G.nz, on);
    } else if (on) {
        g.t[0] = __ldg(ty + idx);
        g.t[1] = __ldg(ty + idx + nyz);
    }
    ld256_if(G.ed + 2 * (int64_t)idx, g.e[0], g.d[0], on);
    ld256_if(G.ed + 2 * (int64_t)(idx + nyz), g.e[1], g.d[1], on);
}

/* trilinear value from the 8 corners, the reference's collapse order and rounding:
 * c(y,z) = lerp(v(0,y,z), v(1,y,z), fx); c0/c1 over y; then z. */
__device__ __forceinline__ float tri8(float v000, float v001, float v010, float v011, float v100,
                                      float v101, float v110, float v111, float fx, float fy,
                                      float fz)
{
    const float c00 = lerp_<true>(v000, v100, fx), c10 = lerp_<true>(v010, v110, fx);
    const float c01 = lerp_<true>(v001, v101, fx), c11 = lerp_<true>(v011, v111, fx);
    const float c0 = lerp_<true>(c00, c10, fy), c1 = lerp_<true>(c01, c11, fy);
    return lerp_<true>(c0, c1, fz);
}

__device__ __forceinline__ float tri_b(const float4 &b0, const float4 &b1, float fx, float fy,
                                       float fz)
{
    /* brick (v[y,z], v[y,z+1], v[y+1,z], v[y+1,z+1]) at x (b0) and x+1 (b1) */
    return tri8(b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, fx, fy, fz);
}

#ifndef VD_PACKED_LERP
#define VD_PACKED_LERP 1
#endif
/* Two reference lerps at once in f32x2: (a*(1-t)) + (b*t) with both products rounded and
 * the sum written as fma(p, one, q) -- ptxas contracts packed mul + add into FFMA2 (see
 * mul2 above) but cannot fold a product into an fma whose multiplier it does not know. */
__device__ __forceinline__ float2 plerp(float2 a, float2 b, float2 omt, float2 t, float2 one)
{
    return __ffma2_rn(__fmul2_rn(a, omt), one, __fmul2_rn(b, t));
}

/* tri_b with the x- and y-collapses paired: (c00, c01) and (c10, c11) are lerps of the
 * z-adjacent corner pairs, then (c0, c1) one more packed lerp; the z-lerp is scalar.
 * Same operations and rounding as tri8. */
__device__ __forceinline__ float tri_bp(const float4 &b0, const float4 &b1, float2 X, float2 OX,
                                        float2 Y, float2 OY, float fz, float omz, float2 one)
{
    const float2 cz0 = plerp(f2(b0.x, b0.y), f2(b1.x, b1.y), OX, X, one);
    const float2 cz1 = plerp(f2(b0.z, b0.w), f2(b1.z, b1.w), OX, X, one);
    const float2 c = plerp(cz0, cz1, OY, Y, one);
    return __fadd_rn(__fmul_rn(c.x, omz), __fmul_rn(c.y, fz));
}

__device__ __forceinline__ float finish_packed(const Gather &g, float q, float dsf, float one)
{
#if VD_PACKED_LERP
    const float2 ONE = f2(one);
    const float2 X = f2(g.fx), OX = f2(__fsub_rn(1.0f, g.fx));
    const float2 Y = f2(g.fy), OY = f2(__fsub_rn(1.0f, g.fy));
    const float omz = __fsub_rn(1.0f, g.fz);
    const float vt = tri_bp(g.t[0], g.t[1], X, OX, Y, OY, g.fz, omz, ONE);
    const float ve = tri_bp(g.e[0], g.e[1], X, OX, Y, OY, g.fz, omz, ONE);
    const float vd = tri_bp(g.d[0], g.d[1], X, OX, Y, OY, g.fz, omz, ONE);
#else
    const float vt = tri_b(g.t[0], g.t[1], g.fx, g.fy, g.fz);
    const float ve = tri_b(g.e[0], g.e[1], g.fx, g.fy, g.fz);
    const float vd = tri_b(g.d[0], g.d[1], g.fx, g.fy, g.fz);
#endif
    const float gterm = __fadd_rn(__fadd_rn(vt, __fmul_rn(q, ve)), __fmul_rn(dsf, vd));
    return g.inb ? gterm : g.pterm;
}

/* One atom of one pose against the plain (n_maps, nx, ny, nz) layout. */
template <bool EXACT, bool ZP = false>
__device__ __forceinline__ float atom_term(const GridView &G, const float *__restrict__ tmap,
                                           const float *__restrict__ emap,
                                           const float *__restrict__ dmap, float q, float dsf,
                                           float pen, float x, float y, float z)
{
    Gather g;
    int idx, zy;
    cell_of(G, x, y, z, pen, g, idx, zy);
    if ((EXACT || ZP) && !g.inb) return g.pterm;  /* ZP (score kernel): out-of-box lanes skip the gathers */
    const int nyz = G.ny * G.nz;
    const float vt = trilerp<true, ZP>(tmap, idx, G.nz, nyz, g.fx, g.fy, g.fz);
    const float ve = trilerp<true, ZP>(emap, idx, G.nz, nyz, g.fx, g.fy, g.fz);
    const float vd = trilerp<true, ZP>(dmap, idx, G.nz, nyz, g.fx, g.fy, g.fz);
    const float gterm = __fadd_rn(__fadd_rn(vt, __fmul_rn(q, ve)), __fmul_rn(dsf, vd));
    return g.inb ? gterm : g.pterm;
}

/* inter of both poses over this sub's atoms; EXACT requires TPP == 1 (atom order).
 * Unpipelined (the score kernel): out-of-box lanes issue no gather requests (~29% of the
 * atoms under cfg1's sampling; 1.543 -> 1.436 ms).  The pipelined GA path keeps unpredicated
 * gathers: its converged populations are mostly in the box (predicating cost it 0.6%).
 * PIPE (packed layout): software-pipelined, the gathers of atom i+TPP are in flight while
 * atom i is interpolated.  That doubles the live gather state (152 vs 94 registers in
 * score_kernel); the score kernel runs unpipelined and covers the latency with its 12
 * resident warps, the GA kernel (register-bound by its other stages anyway) pipelines. */
/* LAY: 0 = both gather paths (run-time choice), 1 = packed grid only, 2 = plain grid only.
 * The kernels are instantiated per layout so that neither path's registers weigh on the
 * other (with both compiled in, the plain path's z-pair gathers took the score kernel from
 * 121 to 168 registers, 1 CTA/SM). */
template <bool EXACT, int NPP, int TPP, bool PIPE, int LAY = 0, bool FLAT = false>
__device__ __forceinline__ void inter2(const LigView &L, const GridView &G, const float2 *S,
                                       int sub, int ia, int ib, double &e0, double &e1)
{
    if (LAY != 2 && G.yz != nullptr && !EXACT) {
        if (FLAT) {
            /* no gather state carried across atoms: inside a loop over pose tiles (the
               persistent score kernel) the carried Gather pair set the register peak
               (92 -> 148 registers for this stage alone) */
            for (int i = ia + sub; i < ib; i += TPP) {
                Gather c0, c1;
                const float2 x = VD_S2(i, 0), y = VD_S2(i, 1), z = VD_S2(i, 2);
                const float4 *tz = type_map(G, __float_as_int(L.atom2[i].y));
                VD_CHK(__float_as_int(L.atom2[i].y) >= 0 && __float_as_int(L.atom2[i].y) < G.n_maps, VD_SITE_MAP);
                int idx0, idx1, zy0, zy1;
                cell_of(G, x.x, y.x, z.x, L.penalty, c0, idx0, zy0);
                cell_of(G, x.y, y.y, z.y, L.penalty, c1, idx1, zy1);
                issue_packed(G, tz, idx0, zy0, c0, true);
                issue_packed(G, tz, idx1, zy1, c1, true);
                const float q = L.atom[i].w, dsf = L.atom2[i].x;
                e0 = __dadd_rn(e0, (double)finish_packed(c0, q, dsf, G.one));
                e1 = __dadd_rn(e1, (double)finish_packed(c1, q, dsf, G.one));
            }
            return;
        }
        const int n = ib;
        int i = ia + sub;
        if (i >= n) return;
        Gather c0, c1;
        {
            const float2 x = VD_S2(i, 0), y = VD_S2(i, 1), z = VD_S2(i, 2);
            const float4 *tz = type_map(G, __float_as_int(L.atom2[i].y));
            VD_CHK(__float_as_int(L.atom2[i].y) >= 0 && __float_as_int(L.atom2[i].y) < G.n_maps, VD_SITE_MAP);
            int idx0, idx1, zy0, zy1;
            cell_of(G, x.x, y.x, z.x, L.penalty, c0, idx0, zy0);
            cell_of(G, x.y, y.y, z.y, L.penalty, c1, idx1, zy1);
            issue_packed(G, tz, idx0, zy0, c0, !PIPE);
            issue_packed(G, tz, idx1, zy1, c1, !PIPE);
        }
        for (; i < n; i += TPP) {
            const int in = i + TPP;
            Gather n0, n1;
            if (!PIPE) {
                const float q = L.atom[i].w, dsf = L.atom2[i].x;
                e0 = __dadd_rn(e0, (double)finish_packed(c0, q, dsf, G.one));
                e1 = __dadd_rn(e1, (double)finish_packed(c1, q, dsf, G.one));
            }
            if (in < n) {
                const float2 x = VD_S2(in, 0), y = VD_S2(in, 1), z = VD_S2(in, 2);
                const float4 *tz = type_map(G, __float_as_int(L.atom2[in].y));
                int idx0, idx1, zy0, zy1;
                cell_of(G, x.x, y.x, z.x, L.penalty, n0, idx0, zy0);
                cell_of(G, x.y, y.y, z.y, L.penalty, n1, idx1, zy1);
                issue_packed(G, tz, idx0, zy0, n0, !PIPE);
                issue_packed(G, tz, idx1, zy1, n1, !PIPE);
            }
            if (PIPE) {
                const float q = L.atom[i].w, dsf = L.atom2[i].x;
                e0 = __dadd_rn(e0, (double)finish_packed(c0, q, dsf, G.one));
                e1 = __dadd_rn(e1, (double)finish_packed(c1, q, dsf, G.one));
            }
            c0 = n0;
            c1 = n1;
        }
        return;
    }
    if constexpr (LAY == 1 && !EXACT) return;
    const float *emap = G.maps + G.mstride * L.elec_map;
    const float *dmap = G.maps + G.mstride * L.desolv_map;
    VD_CHK(L.elec_map >= 0 && L.elec_map < G.n_maps && L.desolv_map >= 0 && L.desolv_map < G.n_maps,
           VD_SITE_MAP);
    /* z-pair loads and the out-of-box early return, atom loop not unrolled: unrolled x2 the
       z-pair gathers raised the score kernel to 168 registers (1 CTA/SM: cfg1 1.41 -> 2.09 ms)
       and cost the GA 7-16%; not unrolled, cfg4 GA 1,297 -> 1,600 ligands/s */
#pragma unroll kPlainUnroll
    for (int i = ia + sub; i < ib; i += TPP) {
        const float4 a = L.atom[i];
        const float2 a2 = L.atom2[i];
        const float *tmap = G.maps + G.mstride * __float_as_int(a2.y);
        VD_CHK(__float_as_int(a2.y) >= 0 && __float_as_int(a2.y) < G.n_maps, VD_SITE_MAP);
        const float2 x = VD_S2(i, 0), y = VD_S2(i, 1), z = VD_S2(i, 2);
        const float t0 = atom_term<EXACT, true>(G, tmap, emap, dmap, a.w, a2.x, L.penalty, x.x, y.x, z.x);
        const float t1 = atom_term<EXACT, true>(G, tmap, emap, dmap, a.w, a2.x, L.penalty, x.y, y.y, z.y);
        e0 = __dadd_rn(e0, (double)t0);
        e1 = __dadd_rn(e1, (double)t1);
    }
}

/* ---- A3: intra ---------------------------------------------------------------- */
__device__ __forceinline__ float pair_exact(float dx, float dy, float dz, bool hb, float4 cf,
                                            float cut2)
{
    const float r2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    if (r2 > cut2) return 0.0f;
    const float r2c = r2 > kMinR2 ? r2 : kMinR2;
    const float inv = __fdiv_rn(1.0f, r2c);
    const float i2 = __fmul_rn(inv, inv), i3 = __fmul_rn(i2, inv), i6 = __fmul_rn(i3, i3);
    const float tail = hb ? __fmul_rn(i3, i2) : i3;
    const float well = __fsub_rn(__fmul_rn(cf.x, i6), __fmul_rn(cf.y, tail));
    const float r = __fsqrt_rn(r2c);
    const double r64 = (double)r;
    const double eps_r = __dadd_rn(kDielA, __ddiv_rn(kDielB, __dadd_rn(1.0, __dmul_rn(kDielK, exp(-__dmul_rn(kLamb, r64))))));
    const float elec = __double2float_rn(__ddiv_rn((double)cf.z, __dmul_rn(r64, eps_r)));
    const float des = __double2float_rn(__dmul_rn((double)cf.w, exp(-__ddiv_rn((double)r2, kDesolvDenom))));
    return __fadd_rn(__fadd_rn(well, elec), des);
}

#ifndef VD_SHARED_RCP
#define VD_SHARED_RCP 0
#endif
#ifndef VD_DESOLV_POLY
#define VD_DESOLV_POLY 0
#endif
/* 2^x for x <= 0 on the FMA pipe (keeps the MUFU pipe for rsqrt/ex2/rcp):
 * n = rint(x) via the 1.5*2^23 magic add, f = x - n in [-1/2, 1/2], degree-5
 * fit of 2^f (max rel err 3e-7), 2^n assembled in the exponent field. */
__device__ __forceinline__ float2 exp2_poly2(float2 x)
{
    x = f2(fmaxf(x.x, -125.0f), fmaxf(x.y, -125.0f));
    const float2 magic = f2(12582912.0f);
    const float2 t = fadd2(x, magic);
    const float2 n = fsub2(t, magic);
    const float2 f = fsub2(x, n);
    float2 p = fma2(f2(0.0012979109305888414f), f, f2(0.009670717641711235f));
    p = fma2(p, f, f2(0.055515434592962265f));
    p = fma2(p, f, f2(0.24022223055362701f));
    p = fma2(p, f, f2(0.6931465268135071f));
    p = fma2(p, f, f2(1.0f));
    const float2 sc = f2(__int_as_float((__float_as_int(t.x) << 23) + 0x3f800000),
                         __int_as_float((__float_as_int(t.y) << 23) + 0x3f800000));
    return fmul2(p, sc);
}

/* FAST pair term for two poses (packed f32x2; MUFU for rsqrt/exp2/rcp).
 *   eps(r) = A + B/(1+K e), e = exp(-lamb r)  =>  elec = qq (1+K e) / (r (A (1+K e) + B)) */
template <bool HB, bool CUT>
__device__ __forceinline__ float2 pair_fast2(float2 dx, float2 dy, float2 dz, float4 cf, float cut2)
{
    const float2 r2 = fma2(dz, dz, fma2(dy, dy, fmul2(dx, dx)));
    const float2 r2c = f2(fmaxf(r2.x, kMinR2), fmaxf(r2.y, kMinR2));
    const float2 rs = f2(mufu_rsq(r2c.x), mufu_rsq(r2c.y));
    const float2 inv = fmul2(rs, rs);
    const float2 r = fmul2(r2c, rs);
    const float2 i2 = fmul2(inv, inv);
    const float2 i3 = fmul2(i2, inv);
    const float2 i6 = fmul2(i3, i3);
    const float2 tail = HB ? fmul2(i3, i2) : i3;
    const float2 well = fma2(f2(cf.x), i6, fmul2(f2(-cf.y), tail));
    const float2 earg = fmul2(r, f2((float)(-kLamb * 1.4426950408889634)));
    const float2 e = f2(mufu_ex2(earg.x), mufu_ex2(earg.y));
    const float2 den = fma2(f2((float)kDielK), e, f2(1.0f));
    const float2 dd = fmul2(r, fma2(f2((float)kDielA), den, f2((float)kDielB)));
#if VD_SHARED_RCP
    /* one MUFU.RCP for both poses: 1/d0 = d1 / (d0 d1), 1/d1 = d0 / (d0 d1).  d = r (A den + B)
       lies in ~[1.2, 2.4e3], so the product cannot overflow; ~3 ulp instead of 1 (the pair
       loop is MUFU-bound: 8 -> 7 MUFU per pose pair) */
    const float qd = mufu_rcp(__fmul_rn(dd.x, dd.y));
    const float2 rc = fmul2(f2(dd.y, dd.x), f2(qd));
#else
    const float2 rc = f2(mufu_rcp(dd.x), mufu_rcp(dd.y));
#endif
    const float2 elec = fmul2(fmul2(f2(cf.z), den), rc);
    const float2 darg = fmul2(r2, f2((float)(-1.4426950408889634 / kDesolvDenom)));
#if VD_DESOLV_POLY
    const float2 des = fmul2(f2(cf.w), exp2_poly2(darg));
#else
    const float2 des = fmul2(f2(cf.w), f2(mufu_ex2(darg.x), mufu_ex2(darg.y)));
#endif
    float2 t = fadd2(fadd2(well, elec), des);
    if (CUT) {
        t.x = r2.x > cut2 ? 0.0f : t.x;
        t.y = r2.y > cut2 ? 0.0f : t.y;
    }
    return t;
}

/* Pair stream [kb, ke) of this sub (stride TPP), deep unroll. */
#ifndef VD_FLAT_UNROLL
#define VD_FLAT_UNROLL 8
#endif
constexpr int kFlatUnroll = VD_FLAT_UNROLL;
template <int NPP, int TPP, bool HB, bool CUT>
__device__ __forceinline__ float2 flat_fast(const float2 *S, int kb, int ke, const float4 *tc,
                                            const int2 *toff, int sub, float cut2)
{
    float2 acc = f2(0.0f);
#pragma unroll kFlatUnroll
    for (int k = kb + sub; k < ke; k += TPP) {
        const float4 c = tc[k];
        const int2 o = toff[k];  /* 3*i, 3*j: pose-tile offsets in units of NPP elements */
        const float2 *Si = S + o.x * NPP, *Sj = S + o.y * NPP;
        acc = fadd2(acc, pair_fast2<HB, CUT>(fsub2(Si[0], Sj[0]), fsub2(Si[NPP], Sj[NPP]),
                                             fsub2(Si[2 * NPP], Sj[2 * NPP]), c, cut2));
    }
    return acc;
}

/* The same sum with i-reuse: each sub walks one contiguous quarter of [kb, ke) (the fast
 * order is row-major inside each hb group, so i stays constant over runs of ~N/2 pairs)
 * and reloads atom i's coordinates only when i changes -- a warp-uniform test, since all
 * lanes of a warp process the same pair.  Per pair that is 3 LDS.64 of the j atom instead
 * of 6: the shared-memory wavefronts of this loop were the largest user of the L1 data
 * pipe the grid gathers also need. */
#ifndef VD_SPLIT_R
#define VD_SPLIT_R 26.0f   /* cost of one atom's gathers in pair-term units (cfg1 sweep) */
#endif
constexpr float kSplitR = VD_SPLIT_R;
#ifndef VD_ROLE_NI8
#define VD_ROLE_NI8 4   /* gather subs per 8 subs in the role-split energy stage */
#endif
#ifndef VD_ROLE_NI_T8
#define VD_ROLE_NI_T8 4   /* gather subs of the 8-sub shapes (3 / 5 measured: see DESIGN) */
#endif
#ifndef VD_INTRA_ROWS
#define VD_INTRA_ROWS 1
#endif
template <int NPP, bool HB, bool CUT>
__device__ __forceinline__ float2 rows_fast(const float2 *S, int kb, int ke, const float4 *tc,
                                            const int2 *toff, unsigned c0, unsigned c1, float cut2)
{
    /* this sub's part [c0, c1) (16.16 fractions) of the range: contiguous, no overlap */
    const int n = ke - kb;
    const int k0 = kb + (int)(((unsigned)n * c0) >> 16), k1 = kb + (int)(((unsigned)n * c1) >> 16);
    float2 acc = f2(0.0f), xi = f2(0.0f), yi = f2(0.0f), zi = f2(0.0f);
    int ci = -1;
#pragma unroll kFlatUnroll
    for (int k = k0; k < k1; ++k) {
        const float4 c = tc[k];
        const int2 o = toff[k];
        if (o.x != ci) {
            ci = o.x;
            xi = S[o.x * NPP];
            yi = S[o.x * NPP + NPP];
            zi = S[o.x * NPP + 2 * NPP];
        }
        const float2 *Sj = S + o.y * NPP;
        acc = fadd2(acc, pair_fast2<HB, CUT>(fsub2(xi, Sj[0]), fsub2(yi, Sj[NPP]),
                                             fsub2(zi, Sj[2 * NPP]), c, cut2));
    }
    return acc;
}

/* Shared-memory pair area (per CTA): the whole list (resident) or one tile. */
struct PairTile {
    float4 *coef;   /* [cap] weight-folded a, b, qq, dsl */
    int *j;         /* [cap] EXACT: packed ij | hb << 31 (reference order) */
    int2 *off;      /* [cap] FAST: 3*i, 3*j -- pose-tile offsets in units of NPP elements, a raw
                       copy of LigView::fij (aliases j) */
    int cap;        /* pairs per buffer; a streamed FAST list has two buffers (coef + cap, off + cap) */
    bool resident;
};

/* Copy pairs [k0, k0 + cnt) of the mode's order into the tile (all CTA threads; caller syncs). */
template <bool EXACT, int NPP>
__device__ __forceinline__ void stage_pairs(const LigView &L, const PairTile &T, int k0, int cnt)
{
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
        VD_CHK(k < T.cap, VD_SITE_TILE);
        if (EXACT) {
            T.coef[k] = __ldg(&L.pcoef[k0 + k]);
            T.j[k] = (int)__ldg(&L.pij[k0 + k]);
            VD_CHK((int)(__ldg(&L.pij[k0 + k]) & 0x7fff) < L.n_atoms &&
                       (int)((__ldg(&L.pij[k0 + k]) >> 15) & 0x7fff) < L.n_atoms, VD_SITE_ATOM);
        } else {
            T.coef[k] = __ldg(&L.fcoef[k0 + k]);
            const int2 w = __ldg(&L.fij[k0 + k]);
            VD_CHK(w.x >= 0 && w.x < 3 * L.n_atoms && w.y >= 0 && w.y < 3 * L.n_atoms, VD_SITE_ATOM);
            T.off[k] = w;
        }
    }
}

/* A resident pair list is staged once per ligand, after stage_topology (same sync). */
template <bool EXACT, int NPP>
__device__ __forceinline__ void stage_resident(const LigView &L, const PairTile &T)
{
    if (T.resident) stage_pairs<EXACT, NPP>(L, T, 0, L.n_pairs);
}

/* FAST resident lists, staged asynchronously: the records are raw copies of the global arrays,
 * so a CTA can start its pose stage (which needs only the topology) while cp.async fills the
 * pair tile; the caller waits (cp_async_wait_all) before the barrier that ends the pose stage.
 * (Staged synchronously, a 32 x 8 CTA waited for ~30 KB of records before the pose stage of
 * its 64 poses: cfg2 screen 960 -> 941 ms.)  The checked build stages synchronously, with the
 * per-record checks of stage_pairs. */
template <int NPP>
__device__ __forceinline__ void stage_resident_async(const LigView &L, const PairTile &T)
{
#ifdef VD_CHECKED
    stage_resident<false, NPP>(L, T);
#else
    if (!T.resident) return;
    for (int k = threadIdx.x; k < L.n_pairs; k += blockDim.x) {
        cp_async16(T.coef + k, L.fcoef + k);
        cp_async8(T.off + k, L.fij + k);
    }
    cp_async_commit();
#endif
}

template <int NPP>
__device__ __forceinline__ void exact_pair(const float2 *S, const PairTile &T, int k, float cut2,
                                           double &acc0, double &acc1)
{
    const uint32_t w = (uint32_t)T.j[k];
    const float4 c = T.coef[k];
    const int i = w & 0x7fff, j = (w >> 15) & 0x7fff;
    const bool hb = w >> 31;
    const float2 xi = VD_S2(i, 0), yi = VD_S2(i, 1), zi = VD_S2(i, 2);
    const float2 xj = VD_S2(j, 0), yj = VD_S2(j, 1), zj = VD_S2(j, 2);
    acc0 = __dadd_rn(acc0, (double)pair_exact(__fsub_rn(xi.x, xj.x), __fsub_rn(yi.x, yj.x),
                                              __fsub_rn(zi.x, zj.x), hb, c, cut2));
    acc1 = __dadd_rn(acc1, (double)pair_exact(__fsub_rn(xi.y, xj.y), __fsub_rn(yi.y, yj.y),
                                              __fsub_rn(zi.y, zj.y), hb, c, cut2));
}

/* intra of both poses over this sub's share of the pairs (all CTA threads must call) */
/* ASYNC (streamed FAST lists): false = one tile buffer, staged through registers (two CTA
 * barriers per tile; the score kernel: its plain-layout gathers are sensitive to the L1 size
 * the shared memory leaves -- a second 6 KB buffer cost cfg4 scoring 9%); true = two buffers
 * filled by cp.async (one barrier per tile, tiles of up to 2,048 pairs; the GA kernels) */
template <bool EXACT, int NPP, int TPP, bool ASYNC = false>
__device__ __forceinline__ void intra2(const LigView &L, const float2 *S, const PairTile &T,
                                       int sub, double &a0, double &a1,
                                       unsigned w0 = ~0u, unsigned w1 = ~0u)
{
    if (w0 == ~0u) {  /* default: equal parts per sub */
        w0 = ((unsigned)sub << 16) / TPP;
        w1 = ((unsigned)(sub + 1) << 16) / TPP;
    }
    const int n = L.n_pairs;
    if (n == 0) return;
    if (EXACT) {
        /* reference lane-8 order (scoring/simd.py:58-86): lane[k & 7] over the
           first 8*floor(n/8) pairs, then a sequential tail, then lanes 0..7 + tail */
        double l0[8], l1[8], tail0 = 0.0, tail1 = 0.0;
#pragma unroll
        for (int l = 0; l < 8; ++l) l0[l] = l1[l] = 0.0;
        const int nblk8 = n & ~7;
        const int step = T.resident ? n : T.cap;
        for (int k0 = 0; k0 < n; k0 += step) {
            const int cnt = min(step, n - k0);
            if (!T.resident) {
                __syncthreads();
                stage_pairs<true, NPP>(L, T, k0, cnt);
                __syncthreads();
            }
            const int cb = min(cnt, max(0, nblk8 - k0));  /* lane-blocked part of this tile */
            for (int kb = 0; kb < cb; kb += 8) {
#pragma unroll
                for (int l = 0; l < 8; ++l) exact_pair<NPP>(S, T, kb + l, L.cut2, l0[l], l1[l]);
            }
            for (int k = cb; k < cnt; ++k) exact_pair<NPP>(S, T, k, L.cut2, tail0, tail1);
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            s0 = __dadd_rn(s0, l0[l]);
            s1 = __dadd_rn(s1, l1[l]);
        }
        a0 = __dadd_rn(s0, tail0);
        a1 = __dadd_rn(s1, tail1);
    } else {
        const bool cut = L.cut2 < INFINITY;
        double s0 = 0.0, s1 = 0.0;
        /* Streamed lists: tiles of T.cap pairs, double-buffered.  The records are raw copies
           of the global arrays, so every thread copies its share of tile t+1 with cp.async
           (no staging registers) while tile t is computed; one CTA barrier per tile makes tile
           t visible and frees the buffer tile t-1 was read from. */
        const int cap = T.resident ? n : T.cap;
        auto issue = [&](int t) {
            const int t0 = t * cap, cnt = min(cap, n - t0);
            const float4 *gc = L.fcoef + t0;
            const int2 *go = L.fij + t0;
            float4 *sc = T.coef + (t & 1) * cap;
            int2 *so = T.off + (t & 1) * cap;
            for (int k = threadIdx.x; k < cnt; k += NPP * TPP) {
                VD_CHK(k < T.cap, VD_SITE_TILE);
                cp_async16(sc + k, gc + k);
                cp_async8(so + k, go + k);
            }
            cp_async_commit();
        };
        /* register-staged single buffer (tiles of kTile pairs): the next tile's records are
           loaded into registers while the current tile is computed */
        constexpr int kPre = ASYNC ? 1 : (kTile + NPP * TPP - 1) / (NPP * TPP);
        float4 pc[kPre];
        int2 pw[kPre];
        auto prefetch = [&](int k0) {
#pragma unroll
            for (int r = 0; r < kPre; ++r) {
                const int k = k0 + (int)threadIdx.x + r * NPP * TPP;
                if ((int)threadIdx.x + r * NPP * TPP < kTile && k < n) {
                    pc[r] = __ldg(&L.fcoef[k]);
                    pw[r] = __ldg(&L.fij[k]);
                }
            }
        };
        if (!T.resident) {
            if (ASYNC) issue(0);
            else prefetch(0);
        }
        for (int t = 0, t0 = 0; t0 < n; ++t, t0 += cap) {
            const int tcnt = min(cap, n - t0);
            const float4 *tc = T.coef;
            const int2 *to = T.off;
            if (!T.resident && !ASYNC) {
                __syncthreads();
#pragma unroll
                for (int r = 0; r < kPre; ++r) {
                    const int k = (int)threadIdx.x + r * NPP * TPP;
                    if (k < tcnt) {
                        VD_CHK(k < T.cap && pw[r].x >= 0 && pw[r].x < 3 * L.n_atoms && pw[r].y >= 0 &&
                                   pw[r].y < 3 * L.n_atoms, VD_SITE_TILE);
                        T.coef[k] = pc[r];
                        T.off[k] = pw[r];
                    }
                }
                __syncthreads();
                if (t0 + cap < n) prefetch(t0 + cap);
            }
            if (!T.resident && ASYNC) {
                cp_async_wait_all();
                __syncthreads();
                if (t0 + cap < n) issue(t + 1);
                tc += (t & 1) * cap;
                to += (t & 1) * cap;
            }
            /* fp32 partials per kTile chunk, flushed to fp64 */
            for (int c0 = 0; c0 < tcnt; c0 += kTile) {
                const int kb = c0, ke = min(tcnt, c0 + kTile);
                const int kh = min(ke, max(kb, L.n_nohb - t0));  /* 12-6 | 12-10 boundary */
#if VD_INTRA_ROWS
                float2 part = cut ? rows_fast<NPP, false, true>(S, kb, kh, tc, to, w0, w1, L.cut2)
                                  : rows_fast<NPP, false, false>(S, kb, kh, tc, to, w0, w1, L.cut2);
                part = fadd2(part, cut ? rows_fast<NPP, true, true>(S, kh, ke, tc, to, w0, w1, L.cut2)
                                       : rows_fast<NPP, true, false>(S, kh, ke, tc, to, w0, w1, L.cut2));
#else
                float2 part = cut ? flat_fast<NPP, TPP, false, true>(S, kb, kh, tc, to, sub, L.cut2)
                                  : flat_fast<NPP, TPP, false, false>(S, kb, kh, tc, to, sub, L.cut2);
                part = fadd2(part, cut ? flat_fast<NPP, TPP, true, true>(S, kh, ke, tc, to, sub, L.cut2)
                                       : flat_fast<NPP, TPP, true, false>(S, kh, ke, tc, to, sub, L.cut2));
#endif
                s0 += (double)part.x;
                s1 += (double)part.y;
            }
        }
        a0 = s0;
        a1 = s1;
    }
}

/* EXACT with TPP = 8 sub-threads per pose pair: the reference's lane-8 fp64 summation
 * (scoring/simd.py:58-86: lane[k & 7] accumulates pairs k < 8*floor(n/8) in order, then a
 * sequential tail, then s = lanes 0..7 in order + tail) with lane l on sub l.  Each lane is
 * the same ordered fp64 chain as in the single-thread path, so the result is bit-identical;
 * the 8 chains run in parallel instead of one thread walking all of them.  The lanes are
 * combined through `red` ([4][TPP][NPP] doubles) by sub 0, which holds a0 / a1 on return
 * (all CTA threads must call). */
template <int NPP, int TPP>
__device__ __forceinline__ void intra_exact_lanes(const LigView &L, const float2 *S, const PairTile &T,
                                                  int sub, double *red, int pp, double &a0, double &a1)
{
    static_assert(TPP == 8, "one reference lane per sub");
    const int n = L.n_pairs;
    double l0 = 0.0, l1 = 0.0, tail0 = 0.0, tail1 = 0.0;
    const int nblk8 = n & ~7;
    const int step = T.resident ? (n > 0 ? n : 1) : T.cap;
    for (int k0 = 0; k0 < n; k0 += step) {
        const int cnt = min(step, n - k0);
        if (!T.resident) {
            __syncthreads();
            stage_pairs<true, NPP>(L, T, k0, cnt);
            __syncthreads();
        }
        const int cb = min(cnt, max(0, nblk8 - k0));  /* lane-blocked part of this tile */
        for (int kb = 0; kb < cb; kb += 8) exact_pair<NPP>(S, T, kb + sub, L.cut2, l0, l1);
        if (sub == 0)
            for (int k = cb; k < cnt; ++k) exact_pair<NPP>(S, T, k, L.cut2, tail0, tail1);
    }
    __syncthreads();  /* red may alias the pair tile or the pose scratch */
    red[(0 * TPP + sub) * NPP + pp] = l0;
    red[(1 * TPP + sub) * NPP + pp] = l1;
    __syncthreads();
    if (sub == 0) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            s0 = __dadd_rn(s0, red[(0 * TPP + l) * NPP + pp]);
            s1 = __dadd_rn(s1, red[(1 * TPP + l) * NPP + pp]);
        }
        a0 = __dadd_rn(s0, tail0);
        a1 = __dadd_rn(s1, tail1);
    }
}

/* inter + intra of both poses (all CTA threads must call) */
template <bool EXACT, int NPP, int TPP, bool PIPE, bool SPLIT, int LAY = 0, bool FLAT = false,
          bool ASYNC = false>
__device__ __forceinline__ void energy2(const LigView &L, const GridView &G, const float2 *S,
                                        const PairTile &T, int sub, double &e0, double &e1,
                                        double &a0, double &a1, double *red = nullptr, int pp = 0,
                                        float split_r = kSplitR)
{
    if constexpr (EXACT && TPP > 1) {
        /* inter: sub 0 alone, atoms in order (a sequential fp64 sum); intra: the 8 reference
           lanes on the 8 subs (intra_exact_lanes).  Sub 0 ends holding all four sums. */
        if (sub == 0) inter2<true, NPP, 1, false, LAY>(L, G, S, 0, 0, L.n_atoms, e0, e1);
        intra_exact_lanes<NPP, TPP>(L, S, T, sub, red, pp, a0, a1);
        return;
    }
    /* SPLIT: the first NI = TPP * VD_ROLE_NI8 / 8 subs gather (L1TEX-bound) while the
       others run the pair sum (MUFU-bound) at the same time, so the two units overlap inside
       one CTA instead of only across CTAs.  Resident pair lists only (the streamed path has
       CTA barriers).  cfg1: 1.603 vs 1.683 ms (NI = 2 of 4); NI = 1 or 3 of 4: 2.23 / 1.76 ms.
       The GA does not split (7,022 vs 8,621 ligands/s): it pipelines its gathers instead. */
    constexpr int NI = TPP == 8 ? VD_ROLE_NI_T8 : (TPP * VD_ROLE_NI8 / 8 > 0 ? TPP * VD_ROLE_NI8 / 8 : 1);
    constexpr int NA = TPP - NI > 0 ? TPP - NI : 1;
    VD_JITTER(100);
    if (SPLIT && !EXACT && TPP >= 4 && NI < TPP && T.resident) {
        /* balance the two roles with the measured cost ratio of one atom's gathers to one
           pair (kSplitR): the pair subs also take the last xa atoms, or the gather subs the
           last px share of the pairs.  cfg1 (40 atoms, 608 pairs), before the in-box-only
           gathers and the packed pose: xa = 6 best of 0/2/4/6/8/10/12 atoms (1.597/1.577/1.560/
           1.545/1.550/1.558/1.567 ms; 10% of the pairs to the gather subs instead: 1.675 ms);
           after them, R = 14/16/18.5/21.7/26/30/36/45 gave 1.553/1.501/1.458/1.435/1.419/
           1.442/1.462/1.484 ms, so R = 26 (xa = 8). */
        const int n = L.n_atoms, np = L.n_pairs;
        const float ex = (float)n - (float)np * (1.0f / split_r);
        const int xa = ex > 0.f ? min(n, (int)(0.5f * ex + 0.5f)) : 0;
        const unsigned px = ex < 0.f ? (unsigned)(-ex * split_r / (2.0f * (float)np) * 65536.0f) : 0u;
        const int acut = n - xa;
        if (sub < NI) {
            inter2<EXACT, NPP, NI, PIPE, LAY, FLAT>(L, G, S, sub, 0, acut, e0, e1);
            if (px) intra2<EXACT, NPP, NA>(L, S, T, sub, a0, a1, 65536u - px + sub * px / NI,
                                           65536u - px + (sub + 1) * px / NI);
        } else {
            const int s = sub - NI;
            intra2<EXACT, NPP, NA>(L, S, T, s, a0, a1, s * (65536u - px) / NA,
                                   (s + 1) * (65536u - px) / NA);
            if (acut < n) inter2<EXACT, NPP, NA, PIPE, LAY, FLAT>(L, G, S, s, acut, n, e0, e1);
        }
        return;
    }
    inter2<EXACT, NPP, TPP, PIPE, LAY, FLAT>(L, G, S, sub, 0, L.n_atoms, e0, e1);
    intra2<EXACT, NPP, TPP, ASYNC>(L, S, T, sub, a0, a1);
}

__device__ __forceinline__ float total32(double inter, double intra, float tors)
{
    return __fadd_rn(__fadd_rn(__double2float_rn(inter), __double2float_rn(intra)), tors);
}

/* Sum per-sub partials (fast mode, TPP > 1) into sub 0; red: double[4][TPP][NPP].
 * EXACT: sub 0 already holds the reference-ordered sums (energy2). */
template <int NPP, int TPP, bool EXACT = false>
__device__ __forceinline__ void reduce_subs(double *red, int pp, int sub, double &e0, double &e1,
                                            double &a0, double &a1)
{
    if (TPP == 1 || EXACT) return;
    VD_JITTER(101);
    __syncthreads();
    red[(0 * TPP + sub) * NPP + pp] = e0;
    red[(1 * TPP + sub) * NPP + pp] = e1;
    red[(2 * TPP + sub) * NPP + pp] = a0;
    red[(3 * TPP + sub) * NPP + pp] = a1;
    __syncthreads();
    if (sub == 0) {
#pragma unroll
        for (int s = 1; s < TPP; ++s) {
            e0 += red[(0 * TPP + s) * NPP + pp];
            e1 += red[(1 * TPP + s) * NPP + pp];
            a0 += red[(2 * TPP + s) * NPP + pp];
            a1 += red[(3 * TPP + s) * NPP + pp];
        }
    }
}

/* Dynamic shared-memory layout of the scoring CTAs. */
struct SmemLayout {
    unsigned topo_atom, topo_atom2, topo_tors, topo_frag, scratch;
    unsigned tile_coef, tile_idx, red, extra, bytes;
    int cap;        /* pairs the tile holds */
    int resident;   /* 1: the whole pair list (n_pairs <= cap) is staged once per ligand */
};

__host__ __device__ inline unsigned align16(unsigned v) { return (v + 15u) & ~15u; }

/* n_pairs: the largest pair list the launch serves (selects resident vs streamed). */
/* A streamed FAST list takes stream_bufs buffers of stream_cap pairs (a multiple of kTile):
 * 1 x kTile, register-staged (the score kernel), or 2 x up to 2,048 filled by cp.async (the
 * GA kernels); see intra2. */
__host__ __device__ inline SmemLayout smem_layout(int n_atoms, int n_tors, int n_frag, int npp,
                                                  int tpp, unsigned extra, int n_pairs,
                                                  int stream_cap = kTile, int stream_bufs = 1)
{
    SmemLayout s;
    unsigned off = align16(8u * 3u * (unsigned)n_atoms * (unsigned)npp);
    s.topo_atom = off;
    off = align16(off + 16u * (unsigned)n_atoms);
    s.topo_atom2 = off;
    off = align16(off + 8u * (unsigned)n_atoms);
    s.topo_tors = off;
    off = align16(off + 16u * (unsigned)n_tors);
    s.topo_frag = off;
    off = align16(off + 4u * (unsigned)n_frag);
    const unsigned scratch_bytes = (tpp > 1) ? 4u * (unsigned)pose_scratch_floats(n_tors) * (unsigned)npp : 0u;
    s.scratch = off;
    off = align16(off + scratch_bytes);
    s.resident = n_pairs <= kResidentPairs;
    s.cap = s.resident ? (((n_pairs > 0 ? n_pairs : 1) + 7) & ~7) : stream_cap;
    const unsigned nbuf = s.resident ? 1u : (unsigned)stream_bufs;
    s.tile_coef = off;
    off += 16u * nbuf * (unsigned)s.cap;
    s.tile_idx = off;
    off = align16(off + 8u * nbuf * (unsigned)s.cap);
    /* the sub reduction reuses the pose scratch (the pose stage is over when it runs;
       the GA syncs before the next tile's pose stage) or a streamed pair tile */
    const unsigned red_bytes = (tpp > 1) ? 8u * 4u * (unsigned)tpp * (unsigned)npp : 0u;
    if (red_bytes <= scratch_bytes) {
        s.red = s.scratch;
    } else if (!s.resident && red_bytes <= 16u * nbuf * (unsigned)s.cap) {  /* the coef buffers */
        s.red = s.tile_coef;
    } else {
        s.red = off;
        off += red_bytes;
    }
    s.extra = align16(off);
    s.bytes = align16(s.extra + extra);
    return s;
}

__device__ __forceinline__ PairTile pair_tile(unsigned char *smem, const SmemLayout &lay)
{
    PairTile T;
    T.coef = reinterpret_cast<float4 *>(smem + lay.tile_coef);
    T.j = reinterpret_cast<int *>(smem + lay.tile_idx);
    T.off = reinterpret_cast<int2 *>(smem + lay.tile_idx);
    T.cap = lay.cap;
    T.resident = lay.resident;
    return T;
}

}  // namespace vd
