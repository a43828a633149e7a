/*
 * vd_ga.cu -- the whole GA of vd/ga.py:180-235 on the device, for a batch of
 * ligands (vd/screening.py:165-244 semantics, ligand i keyed (seed, base+i)).
 *
 * Two device paths, bit-identical to each other (vd_dock_batch picks per group of ligands):
 *   generation-synchronous (fast mode, ligands up to 96 atoms): per generation one
 *     pop_score_kernel launch over all (ligand, pose tile) CTAs and one ga_step_kernel
 *     launch (one CTA per ligand); see the section of that name below
 *   persistent (exact mode, larger ligands, VD_GA_SYNC=0): ga_kernel / ga_team_kernel.
 * Persistent CTAs pull ligands from an atomic work counter (host passes a
 * largest-first order), so ligands of very different sizes balance across
 * the 148 SMs.  One CTA (or team of CTAs) runs one ligand's GA for all generations:
 *   score   thread-per-individual fused pose+inter+intra (vd_device.cuh)
 *   select  block arg-min for the generation best / elites (first index on ties)
 *   breed   thread-per-child tournament, two-point crossover, Gaussian
 *           mutation, quaternion renormalisation (vd/ga.py:120-177)
 * Genes live in a CTA-private double buffer in global memory (L2-resident);
 * only the pose tile, fitness and the per-generation scratch sit in shared
 * memory.  All randomness comes from vd_rng.h's counter-addressed
 * Philox4x64-10 with IEEE-exact transforms, identical to the CPU oracle's.
 */
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

/* Every individual's fast energy is a function of its own genes only.  (r1 shared one
   MUFU.RCP between the two poses of a thread, +0.9% cfg2 screening, but that made a pose's
   energy depend on its pair partner: the elite, re-scored every generation next to a new
   child, changed in the last bits and the generation-best trace rose on most ligands at
   pop 256 x 200, breaking the reference's elitism contract.  Removed.) */
#include "vd_internal.h"
#include "vd_rng.h"

/* Build parts (as in vd_score.cu): VD_PART undefined = one unit;
 * 0 = dispatch, probes and the C entry points; 1..5 = the GA kernels of TPP 1, 2, 4, 8, 16. */
#ifndef VD_PART
#define VD_PART -1
#endif

namespace vd {

struct GaDev {
    int pop, generations, tournament, elitism;
    double cx_rate, mut_rate, sigma_t, sigma_r, sigma_tor;
    double lo[3], hi[3];
};

struct GaOut {
    float *best_total;
    double *best_inter, *best_intra, *best_genes;
    int gstride;
    float *trace;
    int64_t *n_evals;
};

/* block-wide (value, index) arg-min, first index on ties; `skip` flags excluded */
static __device__ int block_argmin(const float *v, const unsigned char *skip, int n, int *s_idx,
                            float *s_val)
{
    float bv = INFINITY;
    int bi = -1;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (skip && skip[i]) continue;
        const float x = v[i];
        if (bi < 0 || x < bv) { bv = x; bi = i; }  /* strided ascending: first min kept */
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_down_sync(0xffffffffu, bv, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_val[warp] = bv; s_idx[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        float v0 = s_val[0];
        int i0 = s_idx[0];
        for (int w = 1; w < nw; ++w) {
            const int oi = s_idx[w];
            const float ov = s_val[w];
            if (oi >= 0 && (i0 < 0 || ov < v0 || (ov == v0 && oi < i0))) { v0 = ov; i0 = oi; }
        }
        s_idx[32] = i0;
    }
    __syncthreads();
    const int r = s_idx[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double dquat_norm(const double *q)
{
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q[0], q[0]), __dmul_rn(q[1], q[1])),
                                          __dmul_rn(q[2], q[2])), __dmul_rn(q[3], q[3])));
}

static __device__ void init_individual(const GaDev &P, int T, int i, uint64_t k0, uint64_t k1, double *g)
{
    const double PI = 3.141592653589793;
    vd_words W = vd_words_at(i, 0, VD_PH_INIT_U, k0, k1);
    for (int a = 0; a < 3; ++a) {
        const double u = vd_u01(vd_words_get(&W, a));
        g[a] = __dadd_rn(P.lo[a], __dmul_rn(__dsub_rn(P.hi[a], P.lo[a]), u));
    }
    double q[4];
    for (int c = 0; c < 4; ++c) q[c] = vd_normal(c, i, 0, VD_PH_INIT_N, k0, k1);
    double n = dquat_norm(q);
    if (n < 1e-12) { q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; n = 1.0; }
    for (int c = 0; c < 4; ++c) g[3 + c] = __ddiv_rn(q[c], n);
    for (int t = 0; t < T; ++t) {
        const double u = vd_u01(vd_words_get(&W, 4 + t));
        g[7 + t] = __dadd_rn(-PI, __dmul_rn(2.0 * PI, u));
    }
}

/* WIDE (ga_step_kernel, 64 registers to spare): the parent loads of four genes are issued
   together; the persistent kernels keep one gene at a time (their register budget) */
template <bool WIDE = false>
static __device__ void breed_child(const GaDev &P, int G, const double *cur, const float *fit, int gen,
                            int c, uint64_t k0, uint64_t k1, double *child)
{
    const int k = P.tournament;
    vd_words W = vd_words_at(c, gen, VD_PH_BREED_U, k0, k1);  /* one Philox block per 4 slots */
    int win[2];
    for (int r = 0; r < 2; ++r) {
        int best = -1;
        for (int j = 0; j < k; ++j) {
            const int idx = (int)vd_below(vd_words_get(&W, r * k + j),
                                          (uint64_t)P.pop);
            VD_CHK(idx >= 0 && idx < P.pop, VD_SITE_POP);
            if (best < 0 || fit[idx] < fit[best]) best = idx;
        }
        win[r] = best;
    }
    const double *p1 = cur + (size_t)win[0] * G, *p2 = cur + (size_t)win[1] * G;
    const bool do_cx = vd_u01(vd_words_get(&W, 2 * k)) < P.cx_rate;
    const int a = (int)vd_below(vd_words_get(&W, 2 * k + 1), (uint64_t)G + 1);
    const int b = (int)vd_below(vd_words_get(&W, 2 * k + 2), (uint64_t)G + 1);
    const int c_lo = min(a, b), c_hi = max(a, b);
    bool mut_rot = false;
    /* vd_u01(w) < rate  <=>  (w >> 11) < ceil(rate * 2^53): (w >> 11) is an integer below 2^53,
       exact as a double, and scaling by 2^-53 is exact, so the integer compare decides every
       word exactly as the fp64 one does (no u64 -> f64 conversion and fp64 multiply per gene);
       WIDE only: in the cfg4 persistent kernel the change of register allocation cost 2% */
    const uint64_t t_mut = !WIDE ? 0ull : P.mut_rate > 0.0 ? __double2ull_ru(fmin(P.mut_rate, 2.0) * 9007199254740992.0) : 0ull;
    /* genes in chunks of 32: first the crossover copy (+0.0, as child + where(mut, z*sigma, 0))
       and the mutation mask, then the normals for the set bits only, so a warp runs the
       normal sampler max-over-lanes(mutations) times rather than once per gene with any
       mutating lane */
    for (int g0 = 0; g0 < G; g0 += 32) {
        const int g1 = min(G, g0 + 32);
        uint32_t mask = 0;
        if (WIDE) {
            /* four genes at a time: their parent loads are issued together, before the flags'
               Philox blocks (one gene at a time, the load latency of every gene was exposed:
               22% of ga_step_kernel's stall samples sat on the copy below) */
            for (int g = g0; g < g1; g += 4) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (g + u < g1) v[u] = ((do_cx && g + u >= c_lo && g + u < c_hi) ? p2 : p1)[g + u];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (g + u < g1) {
                        if ((vd_words_get(&W, 2 * k + 3 + g + u) >> 11) < t_mut) mask |= 1u << (g + u - g0);
                        child[g + u] = __dadd_rn(v[u], 0.0);
                    }
            }
        } else {
            for (int g = g0; g < g1; ++g) {
                const double v = (do_cx && g >= c_lo && g < c_hi) ? p2[g] : p1[g];
                if (vd_u01(vd_words_get(&W, 2 * k + 3 + g)) < P.mut_rate) mask |= 1u << (g - g0);
                child[g] = __dadd_rn(v, 0.0);
            }
        }
        while (mask) {
            const int g = g0 + __ffs(mask) - 1;
            mask &= mask - 1;
            const double v = (do_cx && g >= c_lo && g < c_hi) ? p2[g] : p1[g];
            const double sig = g < 3 ? P.sigma_t : (g < 7 ? P.sigma_r : P.sigma_tor);
            child[g] = __dadd_rn(v, __dmul_rn(vd_normal(g, c, gen, VD_PH_BREED_N, k0, k1), sig));
            mut_rot |= (g >= 3 && g < 7);
        }
    }
    double n = dquat_norm(child + 3);
    const bool bad = n < 1e-9;
    if (bad) {
        for (int q = 3; q < 7; ++q) child[q] = p1[q];
        n = dquat_norm(child + 3);
    }
    if (mut_rot || bad)
        for (int q = 3; q < 7; ++q) child[q] = __ddiv_rn(child[q], n);
}

struct GaLayout {
    SmemLayout base;          /* pose tile + pair tiles (+ reduction) for the largest ligand */
    unsigned off_fit, off_e, off_a, off_taken;
    int team = 1;             /* host: CTAs per ligand (ga_team_kernel when > 1) */
};

/* Per-team global state of ga_team_kernel (one team = `team` CTAs docking one ligand). */
struct GaTeam {
    double *genes;            /* [teams][2][pop][gmax] double-buffered population */
    float *fit;               /* [teams][pop] */
    double *e64, *a64;        /* [teams][pop] */
    unsigned *bar;            /* [teams] arrival counters (zeroed at launch) */
    int *lig;                 /* [teams] the ligand slot the team's leader fetched */
};

#ifndef VD_GA_MINB
#define VD_GA_MINB 1
#endif
#ifndef VD_GA_SPLIT
#define VD_GA_SPLIT 1  /* role-split energy stage (see energy2), as in pop_score_kernel: both GA
                          paths then partition a ligand's fp32 pair sums alike and give
                          bit-identical energies (alone, the split costs the 4-warp persistent
                          CTAs ~19%; they now serve only batches too small for the
                          generation-synchronous path, and ligands it does not cover) */
#endif
#ifndef VD_GA_PIPE
#define VD_GA_PIPE 1   /* software-pipelined grid gathers (see inter2) */
#endif
#ifndef VD_GA_REGS
#define VD_GA_REGS 0   /* >0: register cap per thread (min resident CTAs derived from it) */
#endif
/* both GA paths split the energy stage for 4 and 8 subs (the shapes of ligands up to 96
   atoms); the 16-sub kernels (cfg4: streamed pair lists, which never split) stay without
   the split code, which cost them 780 B of spills */
__host__ __device__ constexpr bool ga_split(int tpp) { return VD_GA_SPLIT != 0 && tpp <= 8; }
/* role-split balance of the GA paths: a GA population sits in the box (every atom gathers),
   so one atom's gathers weigh more pair terms than under cfg1's random poses (kSplitR) */
#ifndef VD_GA_SPLIT_R
#define VD_GA_SPLIT_R 26.0f
#endif
constexpr float kGaSplitR = VD_GA_SPLIT_R;
constexpr int ga_minb(int threads)
{
    return VD_GA_REGS > 0 ? (65536 / (threads * VD_GA_REGS) > 0 ? 65536 / (threads * VD_GA_REGS) : 1)
                          : VD_GA_MINB;
}
/* LAY: 1 packed grid, 2 plain grid */
#ifndef VD_GA_EXACT_MINB
#define VD_GA_EXACT_MINB 2  /* resident CTAs the exact kernels are compiled for (cfg2 exact GA: 1 -> 2 CTAs at 128 registers, 1,017 -> 1,723 ligands/s) */
#endif
template <bool EXACT, int NPP, int TPP, int LAY>
__global__ void __launch_bounds__(NPP *TPP, EXACT ? VD_GA_EXACT_MINB : ga_minb(NPP *TPP)) ga_kernel(GridView Gv, const LigView *__restrict__ ligs,
                                                      const int *__restrict__ order, int count,
                                                      GaDev P, uint64_t seed, int64_t base,
                                                      int *work, double *gene_buf, int gmax,
                                                      GaLayout lay, GaOut out)
{
    constexpr int B = NPP * TPP;
    extern __shared__ __align__(16) unsigned char smem[];
    VD_POISON(smem, lay.base.bytes);
    const int pp = threadIdx.x % NPP, sub = threadIdx.x / NPP;
    float2 *S = reinterpret_cast<float2 *>(smem) + pp;
    const PairTile Tl = pair_tile(smem, lay.base);
    double *red = reinterpret_cast<double *>(smem + lay.base.red);
    float *fit = reinterpret_cast<float *>(smem + lay.off_fit);
    double *e64 = reinterpret_cast<double *>(smem + lay.off_e);
    double *a64 = reinterpret_cast<double *>(smem + lay.off_a);
    unsigned char *taken = smem + lay.off_taken;
    __shared__ int s_lig, s_best;
    __shared__ int s_idx[33];
    __shared__ float s_val[32];
    const int pop = P.pop;
    double *buf0 = gene_buf + (size_t)blockIdx.x * 2 * pop * gmax;
    double *buf1 = buf0 + (size_t)pop * gmax;
    for (;;) {
        if (threadIdx.x == 0) s_lig = atomicAdd(work, 1);
        __syncthreads();
        const int slot = s_lig;
        __syncthreads();
        if (slot >= count) break;
        const int l = order ? order[slot] : slot;
        const LigView L = stage_topology(ligs[l], smem, lay.base.topo_atom, lay.base.topo_atom2,
                                         lay.base.topo_tors, lay.base.topo_frag);
        stage_resident<EXACT, NPP>(L, Tl);
        const int T = L.n_torsions, G = 7 + T;
        const uint64_t k0 = seed, k1 = (uint64_t)(base + l);
        double *cur = buf0, *nxt = buf1;
        for (int i = threadIdx.x; i < pop; i += B) init_individual(P, T, i, k0, k1, cur + (size_t)i * G);
        float best_total = INFINITY;
        bool have = false;
        __syncthreads();
        for (int gen = 0; gen <= P.generations; ++gen) {
            for (int b0 = 0; b0 < pop; b0 += 2 * NPP) {
                /* the tile is free (the previous energy stage's reads ended at
                   reduce_subs' first barrier), the scratch once sub 0 has read the
                   reduction it holds */
                if (TPP > 1 && b0 > 0) __syncthreads();
                const int i0 = b0 + 2 * pp, i1 = i0 + 1;
                build_pose2<NPP, TPP>(L, cur + (size_t)min(i0, pop - 1) * G,
                                      cur + (size_t)min(i1, pop - 1) * G, S, sub,
                                      reinterpret_cast<float *>(smem + lay.base.scratch) + pp, Gv.one);
                if (TPP > 1) __syncthreads();
                double e0 = 0.0, e1 = 0.0, a0 = 0.0, a1 = 0.0;
                energy2<EXACT, NPP, TPP, VD_GA_PIPE != 0, ga_split(TPP), LAY, false, true>(
                    L, Gv, S, Tl, sub, e0, e1, a0, a1, red, pp, kGaSplitR);
                reduce_subs<NPP, TPP, EXACT>(red, pp, sub, e0, e1, a0, a1);
                if (sub == 0) {
                    if (i0 < pop) { e64[i0] = e0; a64[i0] = a0; fit[i0] = total32(e0, a0, L.tors32); }
                    if (i1 < pop) { e64[i1] = e1; a64[i1] = a1; fit[i1] = total32(e1, a1, L.tors32); }
                }
            }
            __syncthreads();
            const int idx = block_argmin(fit, nullptr, pop, s_idx, s_val);
            VD_CHK(idx >= 0 && idx < pop, VD_SITE_POP);
            const float fb = fit[idx];
            const bool better = !have || fb < best_total;  /* strict '<' (vd/ga.py:217) */
            if (better) {
                for (int g = threadIdx.x; g < G; g += B) out.best_genes[(size_t)l * out.gstride + g] = cur[(size_t)idx * G + g];
                if (threadIdx.x == 0) {
                    out.best_total[l] = fb;
                    out.best_inter[l] = e64[idx];
                    out.best_intra[l] = a64[idx];
                }
                best_total = fb;
                have = true;
            }
            if (out.trace && threadIdx.x == 0) out.trace[(size_t)l * (P.generations + 1) + gen] = fb;
            if (gen == P.generations) break;
            /* elites: first `elitism` of a stable ascending sort (vd/ga.py:136-137) */
            for (int i = threadIdx.x; i < pop; i += B) taken[i] = 0;
            __syncthreads();
            for (int e = 0; e < P.elitism; ++e) {
                const int ei = e == 0 ? idx : block_argmin(fit, taken, pop, s_idx, s_val);
                if (threadIdx.x == 0) { taken[ei] = 1; s_best = ei; }
                __syncthreads();
                for (int g = threadIdx.x; g < G; g += B) nxt[(size_t)e * G + g] = cur[(size_t)s_best * G + g];
                __syncthreads();
            }
            VD_JITTER(200);
            for (int c = threadIdx.x; c < pop - P.elitism; c += B)
                breed_child(P, G, cur, fit, gen, c, k0, k1, nxt + (size_t)(P.elitism + c) * G);
            __syncthreads();
            double *t = cur; cur = nxt; nxt = t;
        }
        if (threadIdx.x == 0) out.n_evals[l] = (int64_t)pop * (P.generations + 1);
        __syncthreads();
    }
}

/* Team barrier over the `team` co-resident CTAs of one ligand: arrival counter in global
 * memory, epoch kept per CTA (all CTAs of a team pass the same number of barriers).  The
 * fences order each CTA's global writes (fitness, genes) before its arrival and the team's
 * writes before the reads after the wait. */
__device__ __forceinline__ void team_sync(unsigned *bar, unsigned team, unsigned &epoch)
{
    __syncthreads();
    epoch += team;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (*reinterpret_cast<volatile unsigned *>(bar) < epoch) __nanosleep(100);
        __threadfence();
    }
    __syncthreads();
}

/* ga_kernel with one ligand's population split over a team of `lay.team` CTAs (rank r
 * scores individuals [r*pop/team, (r+1)*pop/team) and breeds children [r*nc/team, ...)),
 * so a batch with few ligands per SM still fills the GPU (BASELINE cfg4 at 8 GPUs: 250
 * ligands per GPU, 148 one-CTA SMs).  Fitness and energies go through per-team global
 * arrays, genes stay in a per-team global double buffer; two team barriers per
 * generation.  Every CTA computes the selection from the full fitness array, so the
 * decisions, the RNG draws (keyed by child index) and the results are bit-identical to
 * ga_kernel's.  Launched cooperatively (all CTAs co-resident). */
template <int NPP, int TPP, int LAY>
__global__ void __launch_bounds__(NPP *TPP) ga_team_kernel(GridView Gv, const LigView *__restrict__ ligs,
                                                           const int *__restrict__ order, int count,
                                                           GaDev P, uint64_t seed, int64_t base,
                                                           int *work, GaTeam tm, int gmax,
                                                           GaLayout lay, GaOut out)
{
    constexpr bool EXACT = false;
    constexpr int B = NPP * TPP;
    extern __shared__ __align__(16) unsigned char smem[];
    VD_POISON(smem, lay.base.bytes);
    const int pp = threadIdx.x % NPP, sub = threadIdx.x / NPP;
    float2 *S = reinterpret_cast<float2 *>(smem) + pp;
    const PairTile Tl = pair_tile(smem, lay.base);
    double *red = reinterpret_cast<double *>(smem + lay.base.red);
    float *fit = reinterpret_cast<float *>(smem + lay.off_fit);
    unsigned char *taken = smem + lay.off_taken;
    __shared__ int s_lig, s_best;
    __shared__ int s_idx[33];
    __shared__ float s_val[32];
    const int pop = P.pop, team = lay.team;
    const int tid = blockIdx.x / team, rank = blockIdx.x % team;
    double *buf0 = tm.genes + (size_t)tid * 2 * pop * gmax, *buf1 = buf0 + (size_t)pop * gmax;
    float *gfit = tm.fit + (size_t)tid * pop;
    double *ge = tm.e64 + (size_t)tid * pop, *ga = tm.a64 + (size_t)tid * pop;
    unsigned *bar = tm.bar + tid;
    unsigned epoch = 0;
    /* scored here: whole pose pairs (2k, 2k+1), as in ga_kernel */
    const int pairs = (pop + 1) / 2;
    const int i_lo = 2 * (rank * pairs / team), i_hi = min(pop, 2 * ((rank + 1) * pairs / team));
    for (;;) {
        if (rank == 0 && threadIdx.x == 0) tm.lig[tid] = atomicAdd(work, 1);
        team_sync(bar, team, epoch);
        if (threadIdx.x == 0) s_lig = *reinterpret_cast<volatile int *>(tm.lig + tid);
        __syncthreads();
        const int slot = s_lig;
        if (slot >= count) break;
        const int l = order ? order[slot] : slot;
        const LigView L = stage_topology(ligs[l], smem, lay.base.topo_atom, lay.base.topo_atom2,
                                         lay.base.topo_tors, lay.base.topo_frag);
        stage_resident<EXACT, NPP>(L, Tl);
        const int T = L.n_torsions, G = 7 + T;
        const int nc = pop - P.elitism;
        const int c_lo = rank * nc / team, c_hi = (rank + 1) * nc / team;  /* bred here */
        const uint64_t k0 = seed, k1 = (uint64_t)(base + l);
        double *cur = buf0, *nxt = buf1;
        for (int i = i_lo + threadIdx.x; i < i_hi; i += B) init_individual(P, T, i, k0, k1, cur + (size_t)i * G);
        float best_total = INFINITY;
        bool have = false;
        __syncthreads();
        for (int gen = 0; gen <= P.generations; ++gen) {
            for (int b0 = i_lo; b0 < i_hi; b0 += 2 * NPP) {
                if (TPP > 1 && b0 > i_lo) __syncthreads();
                const int i0 = b0 + 2 * pp, i1 = i0 + 1;
                build_pose2<NPP, TPP>(L, cur + (size_t)min(i0, i_hi - 1) * G,
                                      cur + (size_t)min(i1, i_hi - 1) * G, S, sub,
                                      reinterpret_cast<float *>(smem + lay.base.scratch) + pp, Gv.one);
                if (TPP > 1) __syncthreads();
                double e0 = 0.0, e1 = 0.0, a0 = 0.0, a1 = 0.0;
                energy2<EXACT, NPP, TPP, VD_GA_PIPE != 0, ga_split(TPP), LAY, false, true>(
                    L, Gv, S, Tl, sub, e0, e1, a0, a1, red, pp, kGaSplitR);
                reduce_subs<NPP, TPP, EXACT>(red, pp, sub, e0, e1, a0, a1);
                if (sub == 0) {
                    if (i0 < i_hi) { ge[i0] = e0; ga[i0] = a0; gfit[i0] = total32(e0, a0, L.tors32); }
                    if (i1 < i_hi) { ge[i1] = e1; ga[i1] = a1; gfit[i1] = total32(e1, a1, L.tors32); }
                }
            }
            team_sync(bar, team, epoch);  /* every slice scored */
            for (int i = threadIdx.x; i < pop; i += B) fit[i] = __ldcg(gfit + i);
            __syncthreads();
            const int idx = block_argmin(fit, nullptr, pop, s_idx, s_val);
            VD_CHK(idx >= 0 && idx < pop, VD_SITE_POP);
            const float fb = fit[idx];
            const bool better = !have || fb < best_total;  /* strict '<' (vd/ga.py:217) */
            if (better) {
                if (rank == 0) {
                    for (int g = threadIdx.x; g < G; g += B)
                        out.best_genes[(size_t)l * out.gstride + g] = __ldcg(cur + (size_t)idx * G + g);
                    if (threadIdx.x == 0) {
                        out.best_total[l] = fb;
                        out.best_inter[l] = __ldcg(ge + idx);
                        out.best_intra[l] = __ldcg(ga + idx);
                    }
                }
                best_total = fb;
                have = true;
            }
            if (rank == 0 && out.trace && threadIdx.x == 0) out.trace[(size_t)l * (P.generations + 1) + gen] = fb;
            if (gen == P.generations) break;
            if (rank == 0) {  /* elites: first `elitism` of a stable ascending sort */
                for (int i = threadIdx.x; i < pop; i += B) taken[i] = 0;
                __syncthreads();
                for (int e = 0; e < P.elitism; ++e) {
                    const int ei = e == 0 ? idx : block_argmin(fit, taken, pop, s_idx, s_val);
                    if (threadIdx.x == 0) { taken[ei] = 1; s_best = ei; }
                    __syncthreads();
                    for (int g = threadIdx.x; g < G; g += B) nxt[(size_t)e * G + g] = __ldcg(cur + (size_t)s_best * G + g);
                    __syncthreads();
                }
            }
            for (int c = c_lo + threadIdx.x; c < c_hi; c += B)
                breed_child(P, G, cur, fit, gen, c, k0, k1, nxt + (size_t)(P.elitism + c) * G);
            team_sync(bar, team, epoch);  /* the next generation is written */
            double *t = cur; cur = nxt; nxt = t;
        }
        if (rank == 0 && threadIdx.x == 0) out.n_evals[l] = (int64_t)pop * (P.generations + 1);
        __syncthreads();
    }
}

/* ---- generation-synchronous GA (fast mode, batches that fill the GPU) ----------------------
 * The persistent kernels above carry the whole GA in one CTA's registers (245 of them: 8-12
 * warps per SM).  For a batch large enough to fill the GPU per generation, every generation
 * is instead two launches over all the batch's ligands:
 *   pop_score_kernel  the score kernel's stages and shape (121 registers, 2 CTAs x 256 threads,
 *                     role-split energy stage) over (ligand, pose tile) CTAs, genes read from
 *                     the batch's population buffer in global memory
 *   ga_step_kernel    one CTA per ligand: generation best, elites, children (the same
 *                     block_argmin / breed_child code and random streams as ga_kernel)
 * Same GA, same streams, and -- since ga_kernel runs a ligand's own sub count and the same role
 * split -- the same energies: both paths are bit-identical (tests/test_gpu_ga.py), each energy
 * a function of the individual's genes alone.  Populations live at pop * gmax doubles per
 * ligand slot, individuals at stride G = 7 + T inside it (as in ga_kernel's buffers). */
template <int NPP, int TPP, int LAY>
__global__ void __launch_bounds__(NPP *TPP) pop_score_kernel(GridView G, const LigView *__restrict__ ligs,
                                                             const int *__restrict__ order,
                                                             int tiles_per_lig, int pop,
                                                             const double *__restrict__ genes, int gmax,
                                                             unsigned smem_bytes, float *__restrict__ fit,
                                                             double *__restrict__ e64,
                                                             double *__restrict__ a64)
{
    extern __shared__ __align__(16) unsigned char smem[];
    VD_POISON(smem, smem_bytes);
    const int pp = threadIdx.x % NPP, sub = threadIdx.x / NPP;
    const int slot = blockIdx.x / tiles_per_lig, tile = blockIdx.x % tiles_per_lig;
    float2 *S = reinterpret_cast<float2 *>(smem) + pp;
    /* the layout of THIS ligand (the launch's shared memory is the largest of its group's
       layouts; one made of the group's maxima would be larger than any of them) */
    const LigView &Lg = ligs[order[slot]];
    const SmemLayout lay = smem_layout(Lg.n_atoms, Lg.n_torsions, Lg.n_frag, NPP, TPP, 0, Lg.n_pairs);
    VD_CHK(lay.bytes <= smem_bytes, VD_SITE_SMEM);
    const PairTile T = pair_tile(smem, lay);
    const LigView L = stage_topology(Lg, smem, lay.topo_atom, lay.topo_atom2,
                                     lay.topo_tors, lay.topo_frag);
    stage_resident_async<NPP>(L, T);  /* lands during the pose stage */
    __syncthreads();
    const int Gn = 7 + L.n_torsions;
    const int i0 = (tile * NPP + pp) * 2, i1 = i0 + 1;
    const double *gb = genes + (size_t)slot * pop * gmax;
    build_pose2<NPP, TPP>(L, gb + (size_t)min(i0, pop - 1) * Gn, gb + (size_t)min(i1, pop - 1) * Gn, S,
                          sub, reinterpret_cast<float *>(smem + lay.scratch) + pp, G.one);
    cp_async_wait_all();  /* this thread's share of the pair records */
    __syncthreads();
    double e0 = 0.0, e1 = 0.0, a0 = 0.0, a1 = 0.0;
    energy2<false, NPP, TPP, false, ga_split(TPP), LAY>(L, G, S, T, sub, e0, e1, a0, a1,
                                               reinterpret_cast<double *>(smem + lay.red), pp, kGaSplitR);
    reduce_subs<NPP, TPP, false>(reinterpret_cast<double *>(smem + lay.red), pp, sub, e0, e1, a0, a1);
    if (sub == 0) {
        const size_t o = (size_t)slot * pop;
        if (i0 < pop) { e64[o + i0] = e0; a64[o + i0] = a0; fit[o + i0] = total32(e0, a0, L.tors32); }
        if (i1 < pop) { e64[o + i1] = e1; a64[o + i1] = a1; fit[o + i1] = total32(e1, a1, L.tors32); }
    }
}

/* One generation's scoring launch.  setup: raise the shared-memory limit and work out the
 * carveout (as many CTAs as fit beside a 32 KB L1 share, see vd_score.cu's launch_t) into
 * *pct; later launches pass it back.  The carveout is a per-function attribute and size
 * buckets share functions, so it is set under a lock right before every launch. */
template <int NPP, int TPP>
cudaError_t launch_pop_t(const GridView &Gv, const LigView *d_ligs, const int *d_order, int count,
                         int pop, const double *genes, int gmax, unsigned bytes, float *fit,
                         double *e64, double *a64, cudaStream_t st, bool setup, int *pct)
{
    auto k = pop_score_kernel<NPP, TPP, 2>;
    if (Gv.yz != nullptr) k = pop_score_kernel<NPP, TPP, 1>;
    static std::mutex mu;
    static int last_pct[2][16];  /* [layout][device]: the carveout last set, + 1 */
    std::lock_guard<std::mutex> lk(mu);
    int dev_now = 0;
    cudaGetDevice(&dev_now);
    int &last = last_pct[Gv.yz != nullptr][dev_now & 15];
    if (setup) {
        last = 0;
        cudaError_t e = vdi::raise_smem_limit((const void *)k, bytes);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        int occ = 0, dev = 0, smem_sm = 0, resv = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NPP * TPP, bytes);
        if (e != cudaSuccess) return e;
        int fit_ctas = (smem_sm - 32 * 1024) / (int)(bytes + resv);
        if (fit_ctas < 2) fit_ctas = std::min(2, smem_sm / (int)(bytes + resv));  /* 2 CTAs beat the L1 share */
        const int want = std::max(1, std::min(occ, fit_ctas));
        *pct = std::min(100, (int)((100LL * want * (bytes + resv) + smem_sm - 1) / smem_sm));
        if (getenv("VD_VERBOSE"))
            fprintf(stderr, "[vd] pop_score_kernel<%d,%d> %d ligands smem=%u ctas/sm=%d carveout=%d%%\n",
                    NPP, TPP, count, bytes, want, *pct);
        return cudaSuccess;
    }
    if (last != *pct + 1) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, *pct);
        if (e != cudaSuccess) return e;
        last = *pct + 1;
    }
    const int tiles = (pop + 2 * NPP - 1) / (2 * NPP);
    k<<<(unsigned)((size_t)count * tiles), NPP * TPP, bytes, st>>>(Gv, d_ligs, d_order, tiles, pop, genes,
                                                                      gmax, bytes, fit, e64, a64);
    ++vdi::g_launches;
    return cudaGetLastError();
}

/* One cooperative launch of the team kernel; `team` CTAs per ligand. */
template <int NPP, int TPP>
cudaError_t launch_ga_team_t(const GridView &Gv, const LigView *d_ligs, const int *d_order,
                                    int count, const GaDev &P, uint64_t seed, int64_t base, int gmax,
                                    const GaLayout &lay, const GaOut &out, cudaStream_t st,
                                    int *d_work, double **team_buf, int *n_ctas)
{
    auto k = ga_team_kernel<NPP, TPP, 2>;
    if (Gv.yz != nullptr) k = ga_team_kernel<NPP, TPP, 1>;
    const unsigned bytes = lay.base.bytes;
    cudaError_t e = vdi::raise_smem_limit((const void *)k, bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NPP * TPP, bytes);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int team = lay.team;
    const int teams = std::max(1, std::min(count, std::max(1, per_sm) * sms / team));
    const int ctas = teams * team;
    /* genes (2 buffers) + fitness + e64 + a64 + barrier + ligand slot per team */
    const size_t gbytes = sizeof(double) * (size_t)teams * 2 * P.pop * gmax;
    const size_t fbytes = sizeof(float) * (size_t)teams * P.pop;
    const size_t ebytes = sizeof(double) * (size_t)teams * P.pop;
    const size_t total = gbytes + fbytes + 2 * ebytes + 2 * sizeof(unsigned) * teams + 64;
    e = cudaMallocAsync((void **)team_buf, total, st);
    if (e != cudaSuccess) return e;
    char *p = reinterpret_cast<char *>(*team_buf);
    GaTeam tm;
    tm.genes = reinterpret_cast<double *>(p);
    tm.e64 = reinterpret_cast<double *>(p + gbytes);
    tm.a64 = reinterpret_cast<double *>(p + gbytes + ebytes);
    tm.fit = reinterpret_cast<float *>(p + gbytes + 2 * ebytes);
    tm.bar = reinterpret_cast<unsigned *>(p + gbytes + 2 * ebytes + fbytes);
    tm.lig = reinterpret_cast<int *>(tm.bar + teams);
    e = cudaMemsetAsync(tm.bar, 0, 2 * sizeof(unsigned) * teams, st);
    if (e != cudaSuccess) return e;
#ifdef VD_CHECKED
    e = cudaMemsetAsync(tm.genes, 0xff, gbytes + fbytes + 2 * ebytes, st);
    if (e != cudaSuccess) return e;
#endif
    GridView gv = Gv;
    GaDev pd = P;
    GaLayout ly = lay;
    GaOut o = out;
    void *args[] = {&gv, (void *)&d_ligs, (void *)&d_order, &count, &pd, &seed, &base, &d_work, &tm,
                    &gmax, &ly, &o};
    e = cudaLaunchCooperativeKernel((const void *)k, dim3(ctas), dim3(NPP * TPP), args, bytes, st);
    ++vdi::g_launches;
    *n_ctas = ctas;
    return e;
}

template <bool EXACT, int NPP, int TPP>
cudaError_t launch_ga_t(const GridView &Gv, const LigView *d_ligs, const int *d_order,
                               int count, const GaDev &P, uint64_t seed, int64_t base, int gmax,
                               const GaLayout &lay, const GaOut &out, cudaStream_t st,
                               int *d_work, double **gene_buf, int *n_ctas)
{
    auto k = ga_kernel<EXACT, NPP, TPP, 2>;  /* plain grid (and every exact launch) */
    if constexpr (!EXACT)
        if (Gv.yz != nullptr) k = ga_kernel<EXACT, NPP, TPP, 1>;  /* packed grid */
    const unsigned bytes = lay.base.bytes;
    cudaError_t e = vdi::raise_smem_limit((const void *)k, bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NPP * TPP, bytes);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ctas = std::max(1, std::min(count, std::max(1, per_sm) * sms));
    e = cudaMallocAsync((void **)gene_buf, sizeof(double) * (size_t)ctas * 2 * P.pop * gmax, st);
    if (e != cudaSuccess) return e;
#ifdef VD_CHECKED
    /* poison the gene double buffers: an individual read before it is written is NaN */
    e = cudaMemsetAsync(*gene_buf, 0xff, sizeof(double) * (size_t)ctas * 2 * P.pop * gmax, st);
    if (e != cudaSuccess) return e;
#endif
    k<<<ctas, NPP * TPP, bytes, st>>>(Gv, d_ligs, d_order, count, P, seed, base, d_work, *gene_buf,
                                      gmax, lay, out);
    ++vdi::g_launches;
    *n_ctas = ctas;
    return cudaGetLastError();
}

template <bool EXACT, int NPP, int TPP>
int occ_t(unsigned bytes, bool packed)
{
    auto k = ga_kernel<EXACT, NPP, TPP, 2>;
    if constexpr (!EXACT)
        if (packed) k = ga_kernel<EXACT, NPP, TPP, 1>;
    if (vdi::raise_smem_limit((const void *)k, bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NPP * TPP, bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm;
}

#define VD_GA_SHAPES(X)                                                     \
    X(1, true, 64, 1) X(1, true, 32, 1) X(1, true, 16, 1)                   \
    X(4, true, 32, 8) X(4, true, 16, 8)                                     \
    X(1, false, 64, 1) X(1, false, 32, 1) X(1, false, 16, 1)                \
    X(2, false, 64, 2) X(2, false, 32, 2) X(2, false, 16, 2)                \
    X(3, false, 64, 4) X(3, false, 32, 4) X(3, false, 16, 4)                \
    X(4, false, 32, 8) X(4, false, 16, 8)                                   \
    X(5, false, 32, 16) X(5, false, 16, 16)
#define VD_GA_TEAM_SHAPES(X) X(4, 32, 8) X(4, 16, 8) X(3, 32, 4) X(3, 16, 4) X(5, 32, 16) X(5, 16, 16)
#define VD_GA_POP_SHAPES(X)                                                 \
    X(1, 64, 1) X(1, 32, 1) X(1, 16, 1) X(3, 64, 4) X(3, 32, 4) X(3, 16, 4) \
    X(4, 32, 8) X(4, 16, 8) X(5, 32, 16) X(5, 16, 16)
/* Every GA launch shape is explicitly instantiated in the build part of its TPP and declared
 * extern in the others (VD_KW_<part> = `template` or `extern template`). */
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
#define VD_GA_INST(P, EX, N, T)                                                                   \
    VD_KW_##P cudaError_t launch_ga_t<EX, N, T>(const GridView &, const LigView *, const int *,  \
                                                int, const GaDev &, uint64_t, int64_t, int,       \
                                                const GaLayout &, const GaOut &, cudaStream_t,    \
                                                int *, double **, int *);                         \
    VD_KW_##P int occ_t<EX, N, T>(unsigned, bool);
#define VD_GA_TEAM_INST(P, N, T)                                                                  \
    VD_KW_##P cudaError_t launch_ga_team_t<N, T>(const GridView &, const LigView *, const int *, \
                                                 int, const GaDev &, uint64_t, int64_t, int,      \
                                                 const GaLayout &, const GaOut &, cudaStream_t,   \
                                                 int *, double **, int *);
#define VD_GA_POP_INST(P, N, T)                                                                   \
    VD_KW_##P cudaError_t launch_pop_t<N, T>(const GridView &, const LigView *, const int *, int, \
                                             int, const double *, int, unsigned,                  \
                                             float *, double *, double *, cudaStream_t, bool,     \
                                             int *);
VD_GA_SHAPES(VD_GA_INST)
VD_GA_TEAM_SHAPES(VD_GA_TEAM_INST)
VD_GA_POP_SHAPES(VD_GA_POP_INST)

#if VD_PART <= 0
/* generation-synchronous GA: dispatch of one scoring launch (false: shape not built) */
bool launch_pop(int npp, int tpp, cudaError_t *err, const GridView &Gv, const LigView *d_ligs,
                const int *d_order, int count, int pop, const double *genes, int gmax,
                unsigned bytes, float *fit, double *e64, double *a64, cudaStream_t st,
                bool setup, int *pct)
{
#define VD_PS(P_, N, T)                                                                          \
    if (npp == N && tpp == T) {                                                                  \
        *err = launch_pop_t<N, T>(Gv, d_ligs, d_order, count, pop, genes, gmax, bytes, fit, e64, \
                                  a64, st, setup, pct);                                          \
        return true;                                                                             \
    }
    VD_GA_POP_SHAPES(VD_PS)
#undef VD_PS
    return false;
}

__global__ void ga_init_kernel(const LigView *__restrict__ ligs, const int *__restrict__ order,
                               GaDev P, uint64_t seed, int64_t base, double *genes, int gmax)
{
    const int slot = blockIdx.x, i = blockIdx.y * blockDim.x + threadIdx.x;  /* x: up to 2^31 - 1 ligands */
    if (i >= P.pop) return;
    const int l = order[slot], T = ligs[l].n_torsions;
    init_individual(P, T, i, seed, (uint64_t)(base + l),
                    genes + (size_t)slot * P.pop * gmax + (size_t)i * (7 + T));
}

/* One GA generation of one ligand per CTA, after its population was scored: the tail of
 * ga_kernel's generation loop (generation best with strict '<', trace, stable elites,
 * thread-per-child breeding into the other buffer). */
__global__ void __launch_bounds__(256, 4) ga_step_kernel(const LigView *__restrict__ ligs,
                                                      const int *__restrict__ order, GaDev P,
                                                      uint64_t seed, int64_t base, int gen,
                                                      const double *__restrict__ cur_all,
                                                      double *__restrict__ nxt_all, int gmax,
                                                      const float *__restrict__ fit_all,
                                                      const double *__restrict__ e_all,
                                                      const double *__restrict__ a_all, GaOut out)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = blockDim.x, pop = P.pop;
    float *fit = reinterpret_cast<float *>(smem);
    unsigned char *taken = smem + 4 * (size_t)pop;
    __shared__ int s_best;
    __shared__ int s_idx[33];
    __shared__ float s_val[32];
    const int slot = blockIdx.x, l = order[slot];
    const int G = 7 + ligs[l].n_torsions;
    const uint64_t k0 = seed, k1 = (uint64_t)(base + l);
    const double *cur = cur_all + (size_t)slot * pop * gmax;
    double *nxt = nxt_all + (size_t)slot * pop * gmax;
    for (int i = threadIdx.x; i < pop; i += B) {
        fit[i] = fit_all[(size_t)slot * pop + i];
        taken[i] = 0;
    }
    __syncthreads();
    const int idx = block_argmin(fit, nullptr, pop, s_idx, s_val);
    VD_CHK(idx >= 0 && idx < pop, VD_SITE_POP);
    const float fb = fit[idx];
    const bool better = gen == 0 || fb < out.best_total[l];  /* strict '<' (vd/ga.py:217) */
    __syncthreads();  /* every thread has read best_total before thread 0 updates it */
    if (better) {
        for (int g = threadIdx.x; g < G; g += B) out.best_genes[(size_t)l * out.gstride + g] = cur[(size_t)idx * G + g];
        if (threadIdx.x == 0) {
            out.best_total[l] = fb;
            out.best_inter[l] = e_all[(size_t)slot * pop + idx];
            out.best_intra[l] = a_all[(size_t)slot * pop + idx];
        }
    }
    if (out.trace && threadIdx.x == 0) out.trace[(size_t)l * (P.generations + 1) + gen] = fb;
    if (gen == P.generations) {
        if (threadIdx.x == 0) out.n_evals[l] = (int64_t)pop * (P.generations + 1);
        return;
    }
    for (int e = 0; e < P.elitism; ++e) {
        const int ei = e == 0 ? idx : block_argmin(fit, taken, pop, s_idx, s_val);
        if (threadIdx.x == 0) { taken[ei] = 1; s_best = ei; }
        __syncthreads();
        for (int g = threadIdx.x; g < G; g += B) nxt[(size_t)e * G + g] = cur[(size_t)s_best * G + g];
        __syncthreads();
    }
    for (int c = threadIdx.x; c < pop - P.elitism; c += B)
        breed_child<true>(P, G, cur, fit, gen, c, k0, k1, nxt + (size_t)(P.elitism + c) * G);
}

cudaError_t launch_ga(bool exact, int npp, int tpp, const GridView &Gv, const LigView *d_ligs,
                      const int *d_order, int count, const GaDev &P, uint64_t seed, int64_t base,
                      int gmax, const GaLayout &lay, const GaOut &out, cudaStream_t st,
                      int *d_work, double **gene_buf, int *n_ctas)
{
    if (!exact && lay.team > 1) {
#define VD_T(P_, N, T)                                                                              \
        if (npp == N && tpp == T)                                                                   \
            return launch_ga_team_t<N, T>(Gv, d_ligs, d_order, count, P, seed, base, gmax, lay, out, \
                                          st, d_work, gene_buf, n_ctas);
        VD_GA_TEAM_SHAPES(VD_T)
#undef VD_T
    }
#define VD_G(P_, EX, N, T)                                                                         \
    if (exact == EX && npp == N && tpp == T)                                                       \
        return launch_ga_t<EX, N, T>(Gv, d_ligs, d_order, count, P, seed, base, gmax, lay, out, st, \
                                     d_work, gene_buf, n_ctas);
    VD_GA_SHAPES(VD_G)
#undef VD_G
    return cudaErrorInvalidConfiguration;
}

int ga_occupancy(bool exact, int npp, int tpp, unsigned bytes, bool packed)
{
#define VD_O(P_, EX, N, T) \
    if (exact == EX && npp == N && tpp == T) return occ_t<EX, N, T>(bytes, packed);
    VD_GA_SHAPES(VD_O)
#undef VD_O
    return 0;
}

/* ---- test probes: the GA's own device draw and operator code on chosen inputs ---- */
__global__ void rng_probe_kernel(int kind, uint64_t k0, uint64_t k1, int phase, int64_t gen,
                                 int64_t n_idx, int n_slot, void *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_idx) return;
    if (kind == 0) {
        vd_words W = vd_words_at(i, gen, phase, k0, k1);
        uint64_t *o = static_cast<uint64_t *>(out) + i * n_slot;
        for (int s = 0; s < n_slot; ++s) o[s] = vd_words_get(&W, s);
    } else {
        double *o = static_cast<double *>(out) + i * n_slot;
        for (int s = 0; s < n_slot; ++s) o[s] = vd_normal(s, i, gen, phase, k0, k1);
    }
}

__global__ void ga_init_probe_kernel(GaDev P, int T, uint64_t k0, uint64_t k1, double *out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P.pop) init_individual(P, T, i, k0, k1, out + (size_t)i * (7 + T));
}

__global__ void ga_breed_probe_kernel(GaDev P, int T, const double *cur, const float *fit, int gen,
                                      uint64_t k0, uint64_t k1, double *out)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int G = 7 + T;
    if (c < P.pop - P.elitism) breed_child(P, G, cur, fit, gen, c, k0, k1, out + (size_t)c * G);
}

}  // namespace vd

using vdi::set_error;

namespace vd {
__global__ void chk_selftest_ga_kernel(int bad) { VD_CHK(bad == 0, VD_SITE_POP); }
}  // namespace vd

namespace vdi {
#if VD_PART == 0
void chk_selftest_ga_part();  /* raises a flag in another build part's word */
#endif
void chk_selftest_ga()
{
    vd::chk_selftest_ga_kernel<<<1, 32>>>(1);
#if VD_PART == 0
    chk_selftest_ga_part();
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
unsigned chk_flags_ga_p1(bool), chk_flags_ga_p2(bool), chk_flags_ga_p3(bool), chk_flags_ga_p4(bool),
    chk_flags_ga_p5(bool);
#endif
unsigned chk_flags_ga(bool clear)
{
    unsigned v = chk_read_own(clear);
#if VD_PART == 0
    v |= chk_flags_ga_p1(clear) | chk_flags_ga_p2(clear) | chk_flags_ga_p3(clear) |
         chk_flags_ga_p4(clear) | chk_flags_ga_p5(clear);
#endif
    return v;
}
}  // namespace vdi

static vd::GaDev ga_dev(const vd_ga_params *p)
{
    vd::GaDev P;
    P.pop = p->pop; P.generations = p->generations; P.tournament = p->tournament;
    P.elitism = p->elitism;
    P.cx_rate = p->cx_rate; P.mut_rate = p->mut_rate;
    P.sigma_t = p->sigma_t; P.sigma_r = p->sigma_r; P.sigma_tor = p->sigma_tor;
    for (int k = 0; k < 3; ++k) { P.lo[k] = p->lo[k]; P.hi[k] = p->hi[k]; }
    return P;
}

extern "C" int vd_debug_rng(int kind, uint64_t seed, uint64_t lig_index, int phase, int64_t gen,
                            int64_t n_idx, int n_slot, void *out)
{
    if ((kind != 0 && kind != 1) || n_idx < 0 || n_slot < 1 || !out) {
        set_error("vd_debug_rng: bad arguments");
        return -1;
    }
    if (n_idx == 0) return 0;
    const size_t bytes = 8u * (size_t)n_idx * n_slot;
    void *d = nullptr;
    VD_CK(cudaMalloc(&d, bytes));
    vd::rng_probe_kernel<<<(unsigned)((n_idx + 127) / 128), 128>>>(kind, seed, lig_index, phase, gen,
                                                                    n_idx, n_slot, d);
    ++vdi::g_launches;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    VD_CK(e);
    return 0;
}

extern "C" int vd_debug_ga_init(const vd_ga_params *p, int n_torsions, uint64_t seed,
                                uint64_t lig_index, double *out)
{
    if (!p || p->pop < 1 || n_torsions < 0 || !out) {
        set_error("vd_debug_ga_init: bad arguments");
        return -1;
    }
    const size_t bytes = sizeof(double) * (size_t)p->pop * (7 + n_torsions);
    double *d = nullptr;
    VD_CK(cudaMalloc((void **)&d, bytes));
    vd::ga_init_probe_kernel<<<(p->pop + 127) / 128, 128>>>(ga_dev(p), n_torsions, seed, lig_index, d);
    ++vdi::g_launches;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    VD_CK(e);
    return 0;
}

extern "C" int vd_debug_ga_breed(const vd_ga_params *p, int n_torsions, const double *cur,
                                 const float *fitness, int gen, uint64_t seed, uint64_t lig_index,
                                 double *children)
{
    if (!p || p->pop < 2 || p->elitism < 0 || p->elitism >= p->pop || p->tournament < 1 ||
        n_torsions < 0 || !cur || !fitness || !children) {
        set_error("vd_debug_ga_breed: bad arguments");
        return -1;
    }
    const int G = 7 + n_torsions, nc = p->pop - p->elitism;
    const size_t pop_bytes = sizeof(double) * (size_t)p->pop * G;
    double *d_cur = nullptr, *d_out = nullptr;
    float *d_fit = nullptr;
    VD_CK(cudaMalloc((void **)&d_cur, pop_bytes));
    VD_CK(cudaMalloc((void **)&d_out, sizeof(double) * (size_t)nc * G));
    VD_CK(cudaMalloc((void **)&d_fit, sizeof(float) * (size_t)p->pop));
    cudaError_t e = cudaMemcpy(d_cur, cur, pop_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_fit, fitness, sizeof(float) * p->pop, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        vd::ga_breed_probe_kernel<<<(nc + 127) / 128, 128>>>(ga_dev(p), n_torsions, d_cur, d_fit, gen,
                                                              seed, lig_index, d_out);
        ++vdi::g_launches;
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(children, d_out, sizeof(double) * (size_t)nc * G, cudaMemcpyDeviceToHost);
    cudaFree(d_cur); cudaFree(d_out); cudaFree(d_fit);
    VD_CK(e);
    return 0;
}

extern "C" int vd_dock_batch(const vd_grid *g, const vd_ligands *s, int first, int count,
                             const vd_ga_params *p, uint64_t seed, int64_t lig_index_base,
                             int mode, float *best_total, double *best_inter, double *best_intra,
                             double *best_genes, int gstride, float *trace, int64_t *n_evals,
                             void *stream)
{
    if (!g || !s || !p || first < 0 || count < 0 || first + count > s->n_ligands) {
        set_error("vd_dock_batch: bad handle or ligand range");
        return -1;
    }
    if (count == 0) return 0;
    if (p->pop < 2 || p->elitism < 0 || p->elitism >= p->pop || p->tournament < 1 ||
        p->generations < 0) {
        set_error("vd_dock_batch: invalid GA parameters");
        return -1;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const bool exact = mode == VD_MODE_EXACT;
    /* ligand views, bucketed by atom count (each bucket gets its own pose-tile
       size and launch shape), largest-first inside a bucket */
    static const int kBucketEdge[] = {24, 32, 48, 64, 96, 128, 192, 256, 1 << 30};
    constexpr int kBuckets = sizeof(kBucketEdge) / sizeof(int);
    std::vector<vd::LigView> views(count);
    /* fast mode, ligands up to 96 atoms with resident pair lists: grouped instead by the
       score-kernel shape each ligand gets on its own (pick_shape, wide) and by the shared-
       memory configuration two of its CTAs need (which sets the L1 share): a ligand's shape,
       and with it the partition of its fp32 pair sums, never depends on its batch mates.
       Groups come after the kBuckets atom-count buckets: key = npp | tpp << 8 | class << 16. */
    std::vector<std::vector<int>> bucket(kBuckets);
    std::vector<int> gkey;
    int tmax = 0;
    for (int l = 0; l < count; ++l) {
        views[l] = s->view(first + l);
        tmax = std::max(tmax, views[l].n_torsions);
        const vd::LigView &V = views[l];
        int sn = 0, stp = 0;
        if (!exact && V.n_atoms <= 96 && V.n_pairs <= vd::kResidentPairs && !getenv("VD_GA_TPP") &&
            vd::pick_shape(V.n_atoms, V.n_pairs, V.n_torsions, false, &sn, &stp, true) == 0) {
            const unsigned two = 2u * (vd::smem_layout(V.n_atoms, V.n_torsions, V.n_frag, sn, stp, 0, V.n_pairs).bytes + 1024u);
            const int cls = two <= 164u * 1024u ? 0 : 1;  /* >= 92 KB of L1 left, or less */
            const int key = sn | (stp << 8) | (cls << 16);
            size_t k = 0;
            while (k < gkey.size() && gkey[k] != key) ++k;
            if (k == gkey.size()) {
                gkey.push_back(key);
                bucket.emplace_back();
            }
            bucket[kBuckets + k].push_back(l);
            continue;
        }
        int b = 0;
        while (V.n_atoms > kBucketEdge[b]) ++b;
        bucket[b].push_back(l);
    }
    /* a small class of a shape joins the shape's other class (the class only sets the L1 share) */
    for (size_t k = 0; k < gkey.size(); ++k)
        for (size_t m = 0; m < gkey.size(); ++m)
            if (m != k && (gkey[m] & 0xffff) == (gkey[k] & 0xffff) && !bucket[kBuckets + k].empty() &&
                bucket[kBuckets + k].size() < 64 && !bucket[kBuckets + m].empty()) {
                auto &src = bucket[kBuckets + k], &dst = bucket[kBuckets + m];
                dst.insert(dst.end(), src.begin(), src.end());
                src.clear();
            }
    const int gmax = 7 + tmax;
    if (gstride < gmax) {
        set_error("vd_dock_batch: gstride smaller than 7 + max torsions");
        return -1;
    }
    const vd::GridView gv = vdi::grid_view(g, s->elec_map, s->desolv_map);
    std::vector<int> order;
    struct Launch {
        int off, cnt, npp, tpp;
        vd::GaLayout lay;
        /* generation-synchronous path (see pop_score_kernel) */
        bool sync = false;
        int s_npp = 0, s_tpp = 0, s_gmax = 0, s_pct = 100;
        unsigned s_bytes = 0;        /* the largest of the group's own layouts */
        double *s_genes = nullptr;   /* [2][cnt][pop][s_gmax] */
        float *s_fit = nullptr;
        double *s_e = nullptr, *s_a = nullptr;
    };
    std::vector<Launch> launches;
    const unsigned extra = (unsigned)p->pop * (4u + 8u + 8u + 1u) + 64u;
    for (int b = 0; b < (int)bucket.size(); ++b) {
        if (bucket[b].empty()) continue;
        auto &v = bucket[b];
        const int key = b >= kBuckets ? gkey[b - kBuckets] : 0;  /* shape group (see above) */
        std::stable_sort(v.begin(), v.end(), [&](int x, int y) {
            return (int64_t)views[x].n_pairs + 4 * views[x].n_atoms >
                   (int64_t)views[y].n_pairs + 4 * views[y].n_atoms;
        });
        int nmax = 1, tb = 0, fb = 0, pmax = 0;
        for (int l : v) {
            nmax = std::max(nmax, views[l].n_atoms);
            tb = std::max(tb, views[l].n_torsions);
            fb = std::max(fb, views[l].n_frag);
            pmax = std::max(pmax, views[l].n_pairs);
        }
        Launch L;
        int npp0;
        if (vd::pick_shape(nmax, pmax, tb, exact, &npp0, &L.tpp)) return -1;
        if (key) L.tpp = (key >> 8) & 0xff;  /* the persistent kernel runs the group's subs too */
        if (!exact)
            if (const char *ov = getenv("VD_GA_TPP")) {  /* tuning override */
                const int v = atoi(ov);
                if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) L.tpp = v;
            }
        /* pose-pairs per CTA: the candidate with most resident warps per SM
           (VD_GA_NPP forces one, for tuning) */
        int best_warps = -1;
        const char *force = getenv("VD_GA_NPP");
        for (int npp : {32, 64, 16}) {  /* ties -> 32 (cfg2 A/B: 6078 vs 5837 ligands/s) */
            if (force && atoi(force) != npp) continue;
            vd::GaLayout lay;
            lay.base = vd::smem_layout(nmax, tb, fb, npp, L.tpp, extra, pmax, vd::kTile, exact ? 1 : 2);
            if (lay.base.bytes > 227u * 1024u) continue;
            if (npp * L.tpp < 32) continue;  /* block_argmin's shuffles need whole warps */
            int warps = vd::ga_occupancy(exact, npp, L.tpp, lay.base.bytes, gv.yz != nullptr) * npp * L.tpp / 32;
            if (npp == 64) warps -= 4;  /* measured: 64 needs clearly more warps to win */
            /* (unlike the score kernel, the GA prefers one 32 x 8 CTA to two 16 x 8 ones at
               the same warps for cfg4: 1239 vs 880 ligands/s -- its per-tile barriers and
               pair-tile streaming are amortised over twice the poses) */
            if (warps > best_warps) {
                best_warps = warps;
                L.npp = npp;
                L.lay = lay;
            }
        }
        if (best_warps <= 0) {
            set_error("vd_dock_batch: population scratch + pose tile exceed shared memory");
            return -1;
        }
        /* streamed pair lists (> kResidentPairs, e.g. cfg4's ~7,600): the largest double-
           buffered tile that keeps the resident CTAs -- one CTA barrier per tile, so a 2,048-
           pair tile means 4 barriers per pose tile for cfg4 instead of 30.  VD_STREAM_CAP
           forces a size (a multiple of 256). */
        if (!L.lay.base.resident && !exact) {
            const int occ0 = vd::ga_occupancy(false, L.npp, L.tpp, L.lay.base.bytes, gv.yz != nullptr);
            int caps[] = {2048, 1024, 512};
            if (const char *ov = getenv("VD_STREAM_CAP")) caps[0] = caps[1] = caps[2] = std::max(256, atoi(ov) & ~255);
            for (int cap : caps) {
                vd::GaLayout lay = L.lay;
                lay.base = vd::smem_layout(nmax, tb, fb, L.npp, L.tpp, extra, pmax, cap, 2);
                if (lay.base.bytes > 227u * 1024u) continue;
                if (vd::ga_occupancy(false, L.npp, L.tpp, lay.base.bytes, gv.yz != nullptr) < occ0) continue;
                L.lay = lay;
                break;
            }
        }
        /* teams: with few ligands per CTA slot (BASELINE cfg4 at 8 GPUs: 250 ligands on 148
           one-CTA SMs, 1.7 waves; a single dock: 1 ligand) a ligand's population is split over
           `team` CTAs so the batch still fills the GPU in whole waves (ga_team_kernel; results
           are bit-identical).
           VD_GA_TEAM=n forces a team size (1 = never split). */
        L.lay.team = 1;
        if (!exact && (L.tpp == 16 || L.tpp == 8 || L.tpp == 4) && (L.npp == 32 || L.npp == 16)) {
            int dev = 0, sms = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int per_sm = std::max(1, vd::ga_occupancy(false, L.npp, L.tpp, L.lay.base.bytes, gv.yz != nullptr));
            const int slots = per_sm * sms;
            /* the whole call's ligands count: the buckets run concurrently, so a small bucket
               of a large batch (cfg2's <= 24-atom tail) must not split (-3% when it did) */
            int team = 1;
            while (team < 8 && (double)count * team / slots < 6.0 && (size_t)count * team < (size_t)(8 * slots)) team *= 2;
            if (const char *ov = getenv("VD_GA_TEAM")) team = std::max(1, std::min(8, atoi(ov)));
            L.lay.team = team;
        }
        if (getenv("VD_VERBOSE"))
            fprintf(stderr, "[vd] ga bucket %d (shape key %#x): %zu ligands, <= %d atoms, npp=%d tpp=%d smem=%u warps/sm=%d team=%d\n",
                    b, key, v.size(), nmax, L.npp, L.tpp, L.lay.base.bytes, best_warps, L.lay.team);
        unsigned off = L.lay.base.extra;
        L.lay.off_e = off;
        off += 8u * p->pop;
        L.lay.off_a = off;
        off += 8u * p->pop;
        L.lay.off_fit = off;
        off += 4u * p->pop;
        L.lay.off_taken = off;
        L.off = (int)order.size();
        L.cnt = (int)v.size();
        /* generation-synchronous path: fast mode, ligands up to 96 atoms (beyond, the
           persistent kernel at 16 subs matches the score kernel), resident pair lists, and
           enough (ligand, tile) CTAs per generation to fill the GPU several times over.
           VD_GA_SYNC=0 keeps the persistent kernels, =1 forces the path where its shape exists. */
        if (key) {
            /* the group's sub count is part of its numerics and fixed; the pose tile is not:
               a batch too small to fill the GPU with its own tile takes smaller ones (a single
               cfg0 dock, pop 100: one 64-pair tile -> four 16-pair CTAs, 2.5 -> 1.6 ms) */
            int sn = key & 0xff;
            const int stp = (key >> 8) & 0xff;
            auto ctas = [&](int n) { return (size_t)L.cnt * ((p->pop + 2 * n - 1) / (2 * n)); };
            while (sn > 16 && ctas(sn) < 2u * 296u) sn /= 2;
            /* ga_step_kernel keeps the fitness and the elite flags in shared memory (5 B per
               individual); populations beyond that stay on the persistent kernels, which
               fail cleanly */
            const unsigned step_bytes = 5u * (unsigned)p->pop + 16u;
            bool want = step_bytes <= 200u * 1024u;
            if (want && step_bytes > 48u * 1024u)
                want = vdi::raise_smem_limit((const void *)vd::ga_step_kernel, step_bytes) == cudaSuccess;
            if (const char *ov = getenv("VD_GA_SYNC")) want = want && atoi(ov) != 0;  /* 0: persistent kernels (A/B, tests) */
            cudaError_t e = cudaSuccess;
            for (int l : v)
                L.s_bytes = std::max(L.s_bytes, vd::smem_layout(views[l].n_atoms, views[l].n_torsions, views[l].n_frag,
                                                               sn, stp, 0, views[l].n_pairs).bytes);
            if (want && vd::launch_pop(sn, stp, &e, gv, nullptr, nullptr, L.cnt, p->pop, nullptr, 0,
                                       L.s_bytes, nullptr, nullptr, nullptr, st, true, &L.s_pct)) {
                VD_CK(e);
                L.sync = true;
                L.s_npp = sn;
                L.s_tpp = stp;
                L.s_gmax = 7 + tb;
            }
        }
        order.insert(order.end(), v.begin(), v.end());
        launches.push_back(L);
    }
    const vd::GaDev P = ga_dev(p);

    const bool dev_out = vdi::is_device_ptr(best_total);
    vd::LigView *d_views = nullptr;
    int *d_order = nullptr, *d_work = nullptr;
    double *gene_buf = nullptr;
    float *d_bt = best_total, *d_tr = trace;
    double *d_be = best_inter, *d_ba = best_intra, *d_bg = best_genes;
    int64_t *d_ne = n_evals;
    const size_t G1 = (size_t)p->generations + 1;
    VD_CK(cudaMallocAsync((void **)&d_views, sizeof(vd::LigView) * count, st));
    VD_CK(cudaMallocAsync((void **)&d_order, sizeof(int) * count, st));
    VD_CK(cudaMallocAsync((void **)&d_work, sizeof(int) * launches.size(), st));
    VD_CK(cudaMemcpyAsync(d_views, views.data(), sizeof(vd::LigView) * count, cudaMemcpyHostToDevice, st));
    VD_CK(cudaMemcpyAsync(d_order, order.data(), sizeof(int) * count, cudaMemcpyHostToDevice, st));
    VD_CK(cudaMemsetAsync(d_work, 0, sizeof(int) * launches.size(), st));
    if (!dev_out) {
        VD_CK(cudaMallocAsync((void **)&d_bt, sizeof(float) * count, st));
        VD_CK(cudaMallocAsync((void **)&d_be, sizeof(double) * count, st));
        VD_CK(cudaMallocAsync((void **)&d_ba, sizeof(double) * count, st));
        VD_CK(cudaMallocAsync((void **)&d_bg, sizeof(double) * count * gstride, st));
        VD_CK(cudaMallocAsync((void **)&d_ne, sizeof(int64_t) * count, st));
        if (trace) VD_CK(cudaMallocAsync((void **)&d_tr, sizeof(float) * count * G1, st));
    }
    VD_CK(cudaMemsetAsync(d_bg, 0, sizeof(double) * count * gstride, st));
    vd::GaOut o;
    o.best_total = d_bt; o.best_inter = d_be; o.best_intra = d_ba; o.best_genes = d_bg;
    o.gstride = gstride; o.trace = d_tr; o.n_evals = d_ne;
    /* Buckets run concurrently, largest atoms first, each on its own stream forked from st:
       a persistent launch ends with a tail of SMs whose CTAs found the work counter empty,
       and the next bucket's CTAs fill them instead of waiting for the whole launch to drain.
       VD_GA_SERIAL=1 keeps the buckets serial on st (A/B). */
    const bool serial = getenv("VD_GA_SERIAL") && atoi(getenv("VD_GA_SERIAL")) != 0;
    std::vector<cudaStream_t> side;
    cudaEvent_t fork = nullptr;
    if (!serial && launches.size() > 1) {
        VD_CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        VD_CK(cudaEventRecord(fork, st));
    }
    std::vector<cudaStream_t> lstream(launches.size(), st);
    /* VD_GA_TIME=1 (tuning): one bucket at a time, host-timed, printed */
    const bool timing = getenv("VD_GA_TIME") != nullptr;
    for (int only = timing ? 0 : -1; only < (timing ? (int)launches.size() : 0); ++only) {
    const auto t_begin = std::chrono::steady_clock::now();
    if (timing) cudaDeviceSynchronize();
    for (int b = (int)launches.size() - 1; b >= 0; --b) {
        if (only >= 0 && b != only) continue;
        Launch &L = launches[b];
        cudaStream_t ls = st;
        if (fork && b != (int)launches.size() - 1) {
            VD_CK(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
            side.push_back(ls);
            VD_CK(cudaStreamWaitEvent(ls, fork, 0));
        }
        lstream[b] = ls;
        if (L.sync) {  /* population buffers + generation 0's individuals */
            const size_t npop = (size_t)L.cnt * p->pop;
            VD_CK(cudaMallocAsync((void **)&L.s_genes, sizeof(double) * 2 * npop * L.s_gmax, ls));
            VD_CK(cudaMallocAsync((void **)&L.s_fit, sizeof(float) * npop, ls));
            VD_CK(cudaMallocAsync((void **)&L.s_e, sizeof(double) * npop, ls));
            VD_CK(cudaMallocAsync((void **)&L.s_a, sizeof(double) * npop, ls));
#ifdef VD_CHECKED
            VD_CK(cudaMemsetAsync(L.s_genes, 0xff, sizeof(double) * 2 * npop * L.s_gmax, ls));
#endif
            vd::ga_init_kernel<<<dim3(L.cnt, (p->pop + 127) / 128), 128, 0, ls>>>(
                d_views, d_order + L.off, P, seed, lig_index_base, L.s_genes, L.s_gmax);
            ++vdi::g_launches;
            VD_CK(cudaGetLastError());
            continue;
        }
        int n_ctas = 0;
        gene_buf = nullptr;
        VD_CK(vd::launch_ga(exact, L.npp, L.tpp, gv, d_views, d_order + L.off, L.cnt, P, seed,
                            lig_index_base, gmax, L.lay, o, ls, d_work + b, &gene_buf, &n_ctas));
        cudaFreeAsync(gene_buf, ls);
    }
    /* generation-synchronous buckets: generation-major over the buckets' streams, so that
       one bucket's launch tails are filled by the others' CTAs */
    for (int gen = 0; gen <= p->generations; ++gen)
        for (int b = (int)launches.size() - 1; b >= 0; --b) {
            Launch &L = launches[b];
            if (!L.sync || (only >= 0 && b != only)) continue;
            const size_t half = (size_t)L.cnt * p->pop * L.s_gmax;
            const double *cur = L.s_genes + (gen & 1) * half;
            double *nxt = L.s_genes + ((gen + 1) & 1) * half;
            cudaError_t e = cudaSuccess;
            vd::launch_pop(L.s_npp, L.s_tpp, &e, gv, d_views, d_order + L.off, L.cnt, p->pop, cur,
                           L.s_gmax, L.s_bytes, L.s_fit, L.s_e, L.s_a, lstream[b], false, &L.s_pct);
            VD_CK(e);
            vd::ga_step_kernel<<<L.cnt, 256, 5u * (unsigned)p->pop + 16u, lstream[b]>>>(
                d_views, d_order + L.off, P, seed, lig_index_base, gen, cur, nxt, L.s_gmax, L.s_fit,
                L.s_e, L.s_a, o);
            ++vdi::g_launches;
            VD_CK(cudaGetLastError());
        }
    for (Launch &L : launches)
        if (L.sync && (only < 0 || &L - launches.data() == only)) {
            const cudaStream_t ls = lstream[&L - launches.data()];
            cudaFreeAsync(L.s_genes, ls);
            cudaFreeAsync(L.s_fit, ls);
            cudaFreeAsync(L.s_e, ls);
            cudaFreeAsync(L.s_a, ls);
        }
    if (timing) {
        cudaDeviceSynchronize();
        const Launch &L = launches[only];
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
        fprintf(stderr, "[vd] ga time: bucket %d %s npp=%d tpp=%d: %d ligands %.1f ms, %.0f M evals/s\n", only,
                L.sync ? "sync" : "persistent", L.sync ? L.s_npp : L.npp, L.sync ? L.s_tpp : L.tpp, L.cnt, ms,
                (double)L.cnt * p->pop * (p->generations + 1) / ms / 1e3);
    }
    }
    for (cudaStream_t ls : side) {  /* join: st waits for every side stream */
        cudaEvent_t done;
        VD_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        VD_CK(cudaEventRecord(done, ls));
        VD_CK(cudaStreamWaitEvent(st, done, 0));
        cudaEventDestroy(done);
        cudaStreamDestroy(ls);  /* released once its work completes */
    }
    if (fork) cudaEventDestroy(fork);
    if (!dev_out) {
        VD_CK(cudaMemcpyAsync(best_total, d_bt, sizeof(float) * count, cudaMemcpyDeviceToHost, st));
        VD_CK(cudaMemcpyAsync(best_inter, d_be, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        VD_CK(cudaMemcpyAsync(best_intra, d_ba, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        VD_CK(cudaMemcpyAsync(best_genes, d_bg, sizeof(double) * count * gstride, cudaMemcpyDeviceToHost, st));
        VD_CK(cudaMemcpyAsync(n_evals, d_ne, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
        if (trace) VD_CK(cudaMemcpyAsync(trace, d_tr, sizeof(float) * count * G1, cudaMemcpyDeviceToHost, st));
        cudaFreeAsync(d_bt, st); cudaFreeAsync(d_be, st); cudaFreeAsync(d_ba, st);
        cudaFreeAsync(d_bg, st); cudaFreeAsync(d_ne, st);
        if (trace) cudaFreeAsync(d_tr, st);
    }
    cudaFreeAsync(d_views, st);
    cudaFreeAsync(d_order, st);
    cudaFreeAsync(d_work, st);
    if (!dev_out) VD_CK(cudaStreamSynchronize(st));
    return 0;
}
#else
}  // namespace vd

namespace vdi {
#define VD_CAT2(a, b) a##b
#define VD_CAT(a, b) VD_CAT2(a, b)
#if VD_PART == 3
}  // namespace vdi
namespace vd {
__global__ void chk_selftest_ga_part_kernel(int bad) { VD_CHK(bad == 0, VD_SITE_CELL); }
}  // namespace vd
namespace vdi {
/* self-test of the per-part flag words: raise a flag in THIS part (read back through part 0) */
void chk_selftest_ga_part()
{
    vd::chk_selftest_ga_part_kernel<<<1, 32>>>(1);
}
#endif
/* this part's check-flag word (see chk_flags_ga in part 0) */
unsigned VD_CAT(chk_flags_ga_p, VD_PART)(bool clear)
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
