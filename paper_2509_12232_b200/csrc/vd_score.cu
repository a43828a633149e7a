/*
 * vd_score.cu -- fused pose + inter + intra scoring kernel.
 *
 * One launch scores P genotypes (or given poses) of ONE ligand:
 * SimdBackend.dock_population / score_many semantics
 * (vd/scoring/simd.py:141-154, 225-240, 277-311) plus the total32 rounding of
 * vd/scoring/__init__.py:345.  A CTA owns 2*NPP poses (NPP pose pairs, TPP
 * threads per pair); see vd_device.cuh for the stage contracts.
 */
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "vd_internal.h"

/* Build parts: the 33 score_kernel instantiations are compiled as five translation units
 * (one per TPP) plus the dispatch, so that `make -j` builds them in parallel:
 *   VD_PART undefined  everything in this one unit
 *   VD_PART 0          dispatch, pose kernels, shape choice; launch_t<> declared extern
 *   VD_PART 1..5       launch_t<*, *, TPP> for TPP = 1, 2, 4, 8, 16 */
#ifndef VD_PART
#define VD_PART -1
#endif

#ifndef VD_SCORE_PIPE
#define VD_SCORE_PIPE 0    /* software-pipelined gathers (see inter2) */
#endif
/* (no min-blocks argument: __launch_bounds__(256, 1) lets ptxas take 140 registers instead
   of 98, which halves the resident CTAs: 2.21 vs 1.56 ms on cfg1) */
#ifndef VD_SCORE_SPLIT
#define VD_SCORE_SPLIT 1   /* role-split energy stage (see energy2) */
#endif

namespace vd {

#ifndef VD_SCORE_PERSIST
#define VD_SCORE_PERSIST 0  /* 1: a CTA walks pose tiles (staging once), flat gathers */
#endif
#ifndef VD_INTER_FLAT
#define VD_INTER_FLAT VD_SCORE_PERSIST
#endif
template <bool EXACT, int NPP, int TPP, int LAY>
__global__ void __launch_bounds__(NPP *TPP) score_kernel(GridView G, LigView Lg,
                                                         const double *__restrict__ genes,
                                                         const float *__restrict__ poses,
                                                         int64_t P, int ngenes, SmemLayout lay,
                                                         double *__restrict__ inter,
                                                         double *__restrict__ intra,
                                                         float *__restrict__ total)
{
    extern __shared__ __align__(16) unsigned char smem[];
    VD_POISON(smem, lay.bytes);
    const int pp = threadIdx.x % NPP, sub = threadIdx.x / NPP;
    float2 *S = reinterpret_cast<float2 *>(smem) + pp;
    const PairTile T = pair_tile(smem, lay);
    const LigView L = stage_topology(Lg, smem, lay.topo_atom, lay.topo_atom2, lay.topo_tors,
                                     lay.topo_frag);
    if (EXACT) stage_resident<EXACT, NPP>(L, T);
    else stage_resident_async<NPP>(L, T);  /* lands during the pose stage */
    __syncthreads();
#if VD_SCORE_PERSIST
    const int64_t n_tiles = (P + 2 * NPP - 1) / (2 * NPP);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        if (tile != blockIdx.x) __syncthreads();  /* tile, scratch and reduction free */
#else
    {
        const int64_t tile = blockIdx.x;
#endif
        const int64_t p0 = (tile * NPP + pp) * 2, p1 = p0 + 1;
        const int64_t q0 = p0 < P ? p0 : P - 1, q1 = p1 < P ? p1 : P - 1;  /* tail: duplicate, drop */
        if (genes) {
            build_pose2<NPP, TPP>(L, genes + q0 * ngenes, genes + q1 * ngenes, S, sub,
                                  reinterpret_cast<float *>(smem + lay.scratch) + pp, G.one);
        } else {
            const int n = L.n_atoms;
            const float *s0 = poses + q0 * 3 * n, *s1 = poses + q1 * 3 * n;
            for (int i = sub; i < n; i += TPP)
#pragma unroll
                for (int c = 0; c < 3; ++c) VD_S2(i, c) = f2(s0[c * n + i], s1[c * n + i]);
        }
        if (!EXACT) cp_async_wait_all();  /* this thread's share of the pair records */
        if (TPP > 1 || !EXACT) __syncthreads();
        double e0 = 0.0, e1 = 0.0, a0 = 0.0, a1 = 0.0;
#ifndef VD_TEST_STAGE
        energy2<EXACT, NPP, TPP, VD_SCORE_PIPE != 0, VD_SCORE_SPLIT != 0, LAY, VD_INTER_FLAT != 0>(
            L, G, S, T, sub, e0, e1, a0, a1, reinterpret_cast<double *>(smem + lay.red), pp);
#else  /* (timing only) the pose stage alone */
        e0 = S[0].x; e1 = S[NPP].y;
#endif
        reduce_subs<NPP, TPP, EXACT>(reinterpret_cast<double *>(smem + lay.red), pp, sub, e0, e1, a0, a1);
        if (sub == 0) {
            if (p0 < P) {
                inter[p0] = e0;
                intra[p0] = a0;
                if (total) total[p0] = total32(e0, a0, L.tors32);
            }
            if (p1 < P) {
                inter[p1] = e1;
                intra[p1] = a1;
                if (total) total[p1] = total32(e1, a1, L.tors32);
            }
        }
    }
}

#if VD_PART <= 0
/* Poses only: the score kernel's pose stage (build_pose2<NPP, TPP>, the same shared tile,
 * scratch and sub-thread split) with the tile written out instead of scored.  TPP = 1 serves
 * vd_pose_genes; TPP = 4 / 8 / 16 are the fast score kernel's shapes (vd_debug_pose_genes). */
template <int NPP, int TPP>
__global__ void __launch_bounds__(NPP *TPP) pose_kernel(LigView Lg, const double *__restrict__ genes,
                                                        int64_t P, int ngenes, SmemLayout lay,
                                                        float one, float *__restrict__ out)
{
    extern __shared__ __align__(16) unsigned char smem[];
    VD_POISON(smem, lay.bytes);
    const int pp = threadIdx.x % NPP, sub = threadIdx.x / NPP;
    const LigView L = stage_topology(Lg, smem, lay.topo_atom, lay.topo_atom2, lay.topo_tors,
                                     lay.topo_frag);
    __syncthreads();
    float2 *S = reinterpret_cast<float2 *>(smem) + pp;
    const int64_t p0 = ((int64_t)blockIdx.x * NPP + pp) * 2, p1 = p0 + 1;
    const int64_t q0 = p0 < P ? p0 : P - 1, q1 = p1 < P ? p1 : P - 1;
    build_pose2<NPP, TPP>(L, genes + q0 * ngenes, genes + q1 * ngenes, S, sub,
                          TPP > 1 ? reinterpret_cast<float *>(smem + lay.scratch) + pp : nullptr, one);
    if (TPP > 1) __syncthreads();
    const int n = L.n_atoms;
    for (int i = sub; i < n; i += TPP)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float2 v = VD_S2(i, c);
            if (p0 < P) out[(p0 * 3 + c) * n + i] = v.x;
            if (p1 < P) out[(p1 * 3 + c) * n + i] = v.y;
        }
}

#endif  /* VD_PART <= 0 */

constexpr unsigned kL1ReserveKB = 32;  /* of the 256 KB L1/shared array, kept as L1 */

#if VD_PART <= 0
/* Launch shape for a ligand: pose pairs per CTA (NPP) and threads per pair (TPP). */
int pick_shape(int n_atoms, int n_pairs, int n_tors, bool exact, int *npp, int *tpp, bool wide)
{
    const unsigned limit = 200 * 1024;
    /* threads per pose pair: more subs for larger ligands, where 12*N bytes of
       shared memory per pose leave few poses (and warps) per SM */
    /* EXACT: 8 subs = the reference's 8 summation lanes (intra_exact_lanes); VD_EXACT_TPP=1
       keeps one thread per pose pair (A/B, and the bitwise cross-check of both paths) */
    /* fast, > 96 atoms: 16 subs (512-thread CTAs at 128 registers, 16 warps per SM where the
       pose tile leaves one CTA per SM): cfg4 GA 336 -> 365 ligands/s, scoring 52.8 -> 54.6 M
       poses/s against 8 subs */
    int t = exact ? 8 : (n_atoms <= 16 ? 1 : (n_atoms <= 96 ? 4 : 16));
    if (exact)
        if (const char *ov = getenv("VD_EXACT_TPP")) t = atoi(ov) == 1 ? 1 : 8;
    if (!exact)
        if (const char *ov = getenv("VD_TPP")) {  /* tuning override: 1, 2 or 4 */
            const int v = atoi(ov);
            if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) t = v;
        }
    int force_npp = 0;
    if (!exact)
        if (const char *ov = getenv("VD_NPP")) force_npp = atoi(ov);  /* tuning override */
    /* wide (the score kernels, 121 registers): when shared memory forces a smaller pose tile,
       more subs keep the CTA at 256 threads, 16 warps per SM with 2 CTAs -- a 59-atom,
       1,451-pair ligand (32 pose pairs per CTA): 315 (32 x 4) -> 422 M poses/s (32 x 8).
       The persistent GA kernels (245 registers) keep 4 subs up to 96 atoms. */
    const bool widen = wide && !exact && t == 4 && !getenv("VD_TPP");
    /* pose pairs per CTA: the largest tile of which 2 CTAs fit beside the L1 share kept
       for the gathers (see launch_t), else the first that fits at all.  cfg1 sweep
       (TPP x NPP, CTAs/SM): 4 x 64 (2) 1.67 ms; 4 x 32 (3) 1.77; 8 x 16 (6) 1.85;
       4 x 128 (1) 1.92; 2 x 64 (2) 1.99.  A bigger tile amortises the shared pair list
       over more poses, so more poses are resident per SM at the same L1 share.  cfg4
       (128 atoms): 8 x 16 (2 CTAs) 45.5 M poses/s vs 8 x 32 (1 CTA, same warps) 39.9 --
       a lone CTA idles the SM at every torsion-chain barrier; 8 x 16 with no L1 share
       (3 CTAs) 28.4: the plain-layout gathers need the L1. */
    const unsigned two_ctas = (228u - kL1ReserveKB) * 1024u / 2u - 1024u;
    for (int pass = 0; pass < 2; ++pass)
        for (int n : {64, 32, 16}) {
            if (force_npp && n != force_npp) continue;
            if (exact && t == 8 && n == 64) continue;  /* 512 threads: beyond the exact kernels' registers */
            if (t == 16 && n == 64) continue;          /* 1,024 threads: not built */
            const int tn = widen ? 256 / n : t;
            const unsigned b = smem_layout(n_atoms, n_tors, 4 * n_atoms, n, tn, 0, n_pairs).bytes;
            /* wide, below 64 pose pairs: two CTAs may take the whole array (28 KB of L1 left):
               32 x 8 with little L1 still beats 16 x 16 (cfg2's 60-atom ligands: 247 M evals/s
               at 16 x 16) */
            const unsigned two = widen && n < 64 ? (228u * 1024u) / 2u - 1024u : two_ctas;
            if (b <= (pass == 0 && !exact ? two : limit)) {
                *npp = n;
                *tpp = tn;
                return 0;
            }
        }
    const std::string why = "ligand too large for the shared-memory pose tile (n_atoms = " +
                            std::to_string(n_atoms) + ")";
    vdi::set_error(why);
    vdi::set_detail(why);
    return -1;
}

#endif  /* VD_PART <= 0 */

template <bool EXACT, int NPP, int TPP>
cudaError_t launch_t(const GridView &G, const LigView &L, const double *genes,
                            const float *poses, int64_t P, int ngenes, double *inter,
                            double *intra, float *total, cudaStream_t st)
{
    const SmemLayout lay = smem_layout(L.n_atoms, L.n_torsions, L.n_frag, NPP, TPP, 0, L.n_pairs);
    auto k = score_kernel<EXACT, NPP, TPP, 2>;  /* plain grid (and every exact launch) */
    if constexpr (!EXACT)
        if (G.yz != nullptr) k = score_kernel<EXACT, NPP, TPP, 1>;  /* packed grid */
    /* the attribute / occupancy set-up below costs ~10 driver calls; a host-buffer batch
       launches once per pipeline chunk, so it is done once per (device, shared-memory size) */
    /* (the function attributes are per kernel: the dynamic shared-memory limit only ever
       grows, and the carveout is re-applied when another shape changed it) */
    struct Setup { int dev; const void *fn; unsigned bytes; int pct; int ctas; };
    /* process-wide (the attributes are): threads scoring different ligands concurrently must
       never lower the limit another thread's launch relies on */
    static std::mutex mu;
    static std::vector<Setup> done_setups;
    struct Carve { int dev; const void *fn; int pct; };
    static std::vector<Carve> last_pct;
    std::lock_guard<std::mutex> lk(mu);
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    int *carve = nullptr;
    for (auto &c : last_pct) if (c.dev == cur_dev && c.fn == (const void *)k) carve = &c.pct;
    if (!carve) { last_pct.push_back({cur_dev, (const void *)k, -1}); carve = &last_pct.back().pct; }
    const char *l1_env = getenv("VD_L1_KB"), *cv_env = getenv("VD_CARVEOUT");
    for (const Setup &x : done_setups)
        if (x.dev == cur_dev && x.fn == (const void *)k && x.bytes == lay.bytes && !l1_env && !cv_env) {
            if (*carve != x.pct) {
                cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, x.pct);
                if (e != cudaSuccess) return e;
                *carve = x.pct;
            }
            const int64_t blocks = std::min<int64_t>((P + 2 * NPP - 1) / (2 * NPP), x.ctas);
            k<<<(unsigned)blocks, NPP * TPP, lay.bytes, st>>>(G, L, genes, poses, P, ngenes, lay,
                                                                inter, intra, total);
            ++vdi::g_launches;
            return cudaGetLastError();
        }
    cudaError_t e = vdi::raise_smem_limit((const void *)k, lay.bytes);
    if (e != cudaSuccess) return e;
    /* Shared-memory carveout: as many CTAs per SM as fit while >= 32 KB of the 256 KB
       L1/shared array stays L1 for the grid gathers (an atom's corners share lines with
       its bonded neighbours').  cfg1 A/B, NPP 32: 1.77 ms at 3 CTAs (63 KB L1) vs 2.00 ms
       at 4 (8 KB L1, the driver's occupancy-maximising default); NPP 64: 1.67 ms at 2. */
    int occ = 0, dev = 0, smem_sm = 0, resv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    /* the occupancy query honours the kernel's CURRENT carveout: after a smaller ligand of the
       same shape had set a low one, a larger ligand was told 1 CTA/SM and ran at half its
       occupancy (31- and 37-atom ligands after a 21-atom one: 657 -> 972 and 502 -> 732 M
       poses/s).  Ask with the carveout at its maximum, then set the one wanted. */
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    *carve = 100;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NPP * TPP, lay.bytes);
    if (e != cudaSuccess) return e;
    int l1_kb = kL1ReserveKB;
    if (const char *w = getenv("VD_L1_KB")) l1_kb = atoi(w);  /* tuning override */
    int fit = (smem_sm - l1_kb * 1024) / (int)(lay.bytes + resv);
    if (fit < 2) fit = std::min(2, smem_sm / (int)(lay.bytes + resv));  /* two CTAs beat the L1 share */
    const int want = std::max(1, std::min(occ, fit));
    int pct = (int)((100LL * want * (lay.bytes + resv) + smem_sm - 1) / smem_sm);
    if (const char *cv = getenv("VD_CARVEOUT")) pct = atoi(cv);  /* tuning override */
    pct = std::min(100, pct);
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    if (e != cudaSuccess) return e;
    *carve = pct;
    /* persistent build: one CTA per resident slot (VD_SCORE_CTAS_PER_SM overrides) */
    int ctas = INT32_MAX;
#if VD_SCORE_PERSIST
    {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int per_sm = want;
        if (const char *c = getenv("VD_SCORE_CTAS_PER_SM")) per_sm = std::max(1, atoi(c));
        ctas = per_sm * sms;
    }
#endif
    if (done_setups.size() < 64) done_setups.push_back({cur_dev, (const void *)k, lay.bytes, pct, ctas});
    const int64_t per_cta = 2 * NPP;
    const int64_t blocks = std::min<int64_t>((P + per_cta - 1) / per_cta, ctas);
    if (getenv("VD_VERBOSE"))
        fprintf(stderr, "[vd] score_kernel<%d,%d,%d> N=%d P=%d smem=%u ctas/sm=%d carveout=%d%%\n",
                (int)EXACT, NPP, TPP, L.n_atoms, L.n_pairs, lay.bytes, want, pct);
    k<<<(unsigned)blocks, NPP * TPP, lay.bytes, st>>>(G, L, genes, poses, P, ngenes, lay, inter,
                                                        intra, total);
    ++vdi::g_launches;
    return cudaGetLastError();
}

/* Every launch shape is explicitly instantiated in the part of its TPP and declared extern
 * in the others (VD_KW_<part> = `template` or `extern template`). */
#if VD_PART < 0 || VD_PART == 1
#define VD_KW_1 template
#else
#define VD_KW_1 extern template
#endif
#if VD_PART < 0 || VD_PART == 2
#define VD_KW_2 template
#else
#define VD_KW_2 extern template
#endif
#if VD_PART < 0 || VD_PART == 3
#define VD_KW_3 template
#else
#define VD_KW_3 extern template
#endif
#if VD_PART < 0 || VD_PART == 4
#define VD_KW_4 template
#else
#define VD_KW_4 extern template
#endif
#if VD_PART < 0 || VD_PART == 5
#define VD_KW_5 template
#else
#define VD_KW_5 extern template
#endif
#define VD_SCORE_INST(P, EX, N, T)                                                              \
    VD_KW_##P cudaError_t launch_t<EX, N, T>(const GridView &, const LigView &, const double *, \
                                             const float *, int64_t, int, double *, double *,   \
                                             float *, cudaStream_t);
#define VD_SCORE_SHAPES(X)                                                  \
    X(1, true, 64, 1) X(1, true, 32, 1) X(1, true, 16, 1)                   \
    X(4, true, 32, 8) X(4, true, 16, 8)                                     \
    X(1, false, 64, 1) X(1, false, 32, 1) X(1, false, 16, 1)                \
    X(2, false, 64, 2) X(2, false, 32, 2) X(2, false, 16, 2)                \
    X(3, false, 64, 4) X(3, false, 32, 4) X(3, false, 16, 4)                \
    X(4, false, 32, 8) X(4, false, 16, 8) X(4, false, 64, 8)                \
    X(5, false, 32, 16) X(5, false, 16, 16)
VD_SCORE_SHAPES(VD_SCORE_INST)

#if VD_PART <= 0
cudaError_t launch_score(int mode, int src, const GridView &G, const LigView &L,
                         const double *genes, const float *poses, int64_t P, int ngenes,
                         double *inter, double *intra, float *total, cudaStream_t st)
{
    const bool exact = mode == VD_MODE_EXACT;
    int npp, tpp;
    if (pick_shape(L.n_atoms, L.n_pairs, L.n_torsions, exact, &npp, &tpp, true)) return cudaErrorInvalidValue;
    if (P <= 0) return cudaSuccess;
    const double *g = src == 0 ? genes : nullptr;
    const float *p = src == 0 ? nullptr : poses;
#define VD_L(P_, EX, N, T) \
    if (exact == EX && npp == N && tpp == T) return launch_t<EX, N, T>(G, L, g, p, P, ngenes, inter, intra, total, st);
    VD_SCORE_SHAPES(VD_L)
#undef VD_L
    return cudaErrorInvalidConfiguration;
}

/* tpp 0: the TPP = 1 pose path of vd_pose_genes; tpp > 0: the fast score kernel's pose-tile
 * shape for that TPP (its NPP from pick_shape), for the bitwise pose test */
cudaError_t launch_pose(const LigView &L, const double *genes, int64_t P, int ngenes, float *out,
                        cudaStream_t st, int tpp_force)
{
    int npp, tpp;
    if (tpp_force > 0) {
        if (pick_shape(L.n_atoms, L.n_pairs, L.n_torsions, false, &npp, &tpp)) return cudaErrorInvalidValue;
        tpp = tpp_force;
        if (tpp == 16 && npp == 64) npp = 32;  /* 64 x 16 is not built */
        const unsigned b = smem_layout(L.n_atoms, L.n_torsions, L.n_frag, npp, tpp, 0, 0).bytes;
        if (b > 200u * 1024u) return cudaErrorInvalidValue;
    } else if (pick_shape(L.n_atoms, 0, L.n_torsions, true, &npp, &tpp)) {
        return cudaErrorInvalidValue;
    }
    if (P <= 0) return cudaSuccess;
    const SmemLayout lay = smem_layout(L.n_atoms, L.n_torsions, L.n_frag, npp, tpp, 0, 0);
    const size_t smem = lay.bytes;
    const int64_t blocks = (P + 2 * npp - 1) / (2 * npp);
    cudaError_t e = cudaErrorInvalidConfiguration;
#define VD_P(N, T)                                                                                \
    if (npp == N && tpp == T) {                                                                   \
        e = vdi::raise_smem_limit((const void *)pose_kernel<N, T>, (unsigned)smem);                \
        if (e == cudaSuccess)                                                                     \
            pose_kernel<N, T><<<(unsigned)blocks, N * T, smem, st>>>(L, genes, P, ngenes, lay,    \
                                                                     1.0f /* run-time: see xadd2 */, out); \
    }
    VD_P(64, 1) else VD_P(32, 1) else VD_P(16, 1)
    else VD_P(64, 4) else VD_P(32, 4) else VD_P(16, 4)
    else VD_P(64, 8) else VD_P(32, 8) else VD_P(16, 8)
    else VD_P(32, 16) else VD_P(16, 16)
#undef VD_P
    if (e != cudaSuccess) return e;
    ++vdi::g_launches;
    return cudaGetLastError();
}

}  // namespace vd

namespace vd {
__global__ void chk_selftest_score_kernel(int bad) { VD_CHK(bad == 0, VD_SITE_TILE); }
}  // namespace vd

namespace vdi {
#if VD_PART == 0
void chk_selftest_score_part();  /* raises a flag in another build part's word */
#endif
void chk_selftest_score()
{
    vd::chk_selftest_score_kernel<<<1, 32>>>(1);
#if VD_PART == 0
    chk_selftest_score_part();
#endif
}

/* the check-flag word is per translation unit: every build part reads its own, part 0 (or
   the single unit) ORs them */
static unsigned chk_read_own(bool clear)
{
#ifdef VD_CHECKED
    unsigned v = 0;
    cudaMemcpyFromSymbol(&v, vd::g_vd_chk_flags, sizeof v);
    if (clear) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(vd::g_vd_chk_flags, &z, sizeof z);
    }
    return v;
#else
    (void)clear;
    return 0;
#endif
}
#if VD_PART == 0
unsigned chk_flags_score_p1(bool), chk_flags_score_p2(bool), chk_flags_score_p3(bool), chk_flags_score_p4(bool),
    chk_flags_score_p5(bool);
#endif
unsigned chk_flags_score(bool clear)
{
    unsigned v = chk_read_own(clear);
#if VD_PART == 0
    v |= chk_flags_score_p1(clear) | chk_flags_score_p2(clear) | chk_flags_score_p3(clear) |
         chk_flags_score_p4(clear) | chk_flags_score_p5(clear);
#endif
    return v;
}
}  // namespace vdi
#else
}  // namespace vd

namespace vdi {
#define VD_CAT2(a, b) a##b
#define VD_CAT(a, b) VD_CAT2(a, b)
#if VD_PART == 3
}  // namespace vdi
namespace vd {
__global__ void chk_selftest_score_part_kernel(int bad) { VD_CHK(bad == 0, VD_SITE_SMEM); }
}  // namespace vd
namespace vdi {
/* self-test of the per-part flag words: raise a flag in THIS part (read back through part 0) */
void chk_selftest_score_part()
{
    vd::chk_selftest_score_part_kernel<<<1, 32>>>(1);
}
#endif
/* this part's check-flag word (see chk_flags_score in part 0) */
unsigned VD_CAT(chk_flags_score_p, VD_PART)(bool clear)
{
#ifdef VD_CHECKED
    unsigned v = 0;
    cudaMemcpyFromSymbol(&v, vd::g_vd_chk_flags, sizeof v);
    if (clear) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(vd::g_vd_chk_flags, &z, sizeof z);
    }
    return v;
#else
    (void)clear;
    return 0;
#endif
}
}  // namespace vdi
#endif  /* VD_PART <= 0 */
