/*
 * vd_ga_oracle.c -- CPU restatement of the GA (TEST INFRASTRUCTURE ONLY;
 * see vd_oracle.c for who may load it).
 *
 * Operators follow vd/ga.py line by line:
 *   init_population  ga.py:90-109   t ~ U(box), q = N(0,1)^4 normalised
 *                                   (degenerate -> identity), theta ~ U(-pi, pi)
 *   next_generation  ga.py:120-177  stable-argsort elites, tournament argmin
 *                                   (first index on ties), two sorted cuts in
 *                                   [0, G] with p2 in [c0, c1), per-gene
 *                                   mutation `child + where(mut, z*sigma, 0.0)`,
 *                                   quaternion renormalised when mutated or
 *                                   degenerate (< 1e-9 -> parent 1's rotation)
 *   dock             ga.py:180-235  G+1 scorings, best with strict '<', trace
 *                                   = per-generation best
 * Only the random stream differs from the reference (numpy's sequential
 * Generator cannot run data-parallel): every draw is addressed by counter
 * through or_rng.c, the oracle's own restatement of the counter map and
 * transforms.  No product source is compiled in here:
 * the device GA is checked against this independent stream bit for bit.
 *
 * Arithmetic: the reference's numpy float64 element-wise operations are
 * single IEEE operations; -ffp-contract=off keeps them unfused.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "vd_oracle.h"
#include "or_rng.h"

typedef struct {
    int pop, generations, tournament, elitism;
    double cx_rate, mut_rate, sigma_t, sigma_r, sigma_tor;
    double lo[3], hi[3];
} or_ga_params;

typedef struct {
    int64_t children, crossovers, gene_mutations, genes_seen;
} or_ga_counts;

void or_init_population(const or_ga_params *P, int n_torsions, uint64_t k0, uint64_t k1,
                        double *pop /* (pop, 7+T) */)
{
    const int G = 7 + n_torsions;
    const double PI = 3.141592653589793;
    const or_rng_key key = {k0, k1};
    for (int i = 0; i < P->pop; ++i) {
        double *g = pop + (size_t)i * G;
        /* t = lo + (hi - lo) * U (ga.py:101-102); slots 0-2 of the init uniforms */
        for (int a = 0; a < 3; ++a) {
            double u = or_rng_uniform(or_rng_word(&key, OR_PH_INIT_U, 0, i, a));
            g[a] = P->lo[a] + (P->hi[a] - P->lo[a]) * u;
        }
        /* q = N(0,1)^4 / |q| (ga.py:103-106) */
        double q[4];
        for (int c = 0; c < 4; ++c) q[c] = or_rng_normal(&key, OR_PH_INIT_N, 0, i, c);
        double n = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        if (n < 1e-12) { q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; n = 1.0; }
        for (int c = 0; c < 4; ++c) g[3 + c] = q[c] / n;
        /* theta = -pi + 2 pi U (ga.py:107-108); slots 4.. */
        for (int t = 0; t < n_torsions; ++t) {
            double u = or_rng_uniform(or_rng_word(&key, OR_PH_INIT_U, 0, i, 4 + t));
            g[7 + t] = -PI + (2.0 * PI) * u;
        }
    }
}

static double quat_norm(const double *q)
{
    return sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
}

/* One child of generation `gen` (ga.py:139-174 for a single row). */
void or_breed_child(const or_ga_params *P, int G, const double *cur, const double *fit,
                    int gen, int c, uint64_t k0, uint64_t k1, double *child, or_ga_counts *cnt)
{
    const int k = P->tournament;
    const or_rng_key key = {k0, k1};
#define BREED_WORD(slot) or_rng_word(&key, OR_PH_BREED_U, gen, c, (slot))
    int win[2];
    for (int r = 0; r < 2; ++r) {
        int best = -1;
        for (int j = 0; j < k; ++j) {
            int idx = (int)or_rng_below(BREED_WORD(r * k + j), (uint64_t)P->pop);
            if (best < 0 || fit[idx] < fit[best]) best = idx;
        }
        win[r] = best;
    }
    const double *p1 = cur + (size_t)win[0] * G, *p2 = cur + (size_t)win[1] * G;
    int do_cx = or_rng_uniform(BREED_WORD(2 * k)) < P->cx_rate;
    int a = (int)or_rng_below(BREED_WORD(2 * k + 1), (uint64_t)G + 1);
    int b = (int)or_rng_below(BREED_WORD(2 * k + 2), (uint64_t)G + 1);
    int c_lo = a < b ? a : b, c_hi = a < b ? b : a;
    int mut_rot = 0;
    for (int g = 0; g < G; ++g) {
        double v = (do_cx && g >= c_lo && g < c_hi) ? p2[g] : p1[g];
        int mut = or_rng_uniform(BREED_WORD(2 * k + 3 + g)) < P->mut_rate;
        double noise = 0.0;
        if (mut) {
            double sig = g < 3 ? P->sigma_t : (g < 7 ? P->sigma_r : P->sigma_tor);
            noise = or_rng_normal(&key, OR_PH_BREED_N, gen, c, g) * sig;
            if (g >= 3 && g < 7) mut_rot = 1;
            if (cnt) cnt->gene_mutations++;
        }
        child[g] = v + noise;
    }
#undef BREED_WORD
    double n = quat_norm(child + 3);
    int bad = n < 1e-9;
    if (bad) {
        memcpy(child + 3, p1 + 3, 4 * sizeof(double));
        n = quat_norm(child + 3);
    }
    if (mut_rot || bad)
        for (int q = 3; q < 7; ++q) child[q] = child[q] / n;
    if (cnt) {
        cnt->children++;
        cnt->crossovers += do_cx;
        cnt->genes_seen += G;
    }
}

/* Elites: first `E` of a stable ascending argsort of fitness. */
static void elites_of(const double *fit, int pop, int E, int *out)
{
    for (int e = 0; e < E; ++e) {
        int best = -1;
        for (int i = 0; i < pop; ++i) {
            int taken = 0;
            for (int q = 0; q < e; ++q) taken |= out[q] == i;
            if (taken) continue;
            if (best < 0 || fit[i] < fit[best]) best = i;
        }
        out[e] = best;
    }
}

void or_next_generation(const or_ga_params *P, int n_torsions, const double *cur,
                        const double *fit, int gen, uint64_t k0, uint64_t k1, double *next,
                        or_ga_counts *cnt)
{
    const int G = 7 + n_torsions, E = P->elitism;
    int *el = (int *)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
    elites_of(fit, P->pop, E, el);
    for (int e = 0; e < E; ++e) memcpy(next + (size_t)e * G, cur + (size_t)el[e] * G, G * sizeof(double));
    for (int c = 0; c < P->pop - E; ++c)
        or_breed_child(P, G, cur, fit, gen, c, k0, k1, next + (size_t)(E + c) * G, cnt);
    free(el);
}

/* Full dock of one ligand (ga.py:180-235). */
int or_dock(const or_ligand *L, const or_ga_params *P, uint64_t seed, uint64_t lig_index,
            float tors32, double *best_genes, float *best_total, double *best_inter,
            double *best_intra, float *trace, int64_t *n_evals)
{
    const int T = L->n_torsions, G = 7 + T, pop = P->pop, n = L->n_atoms;
    double *cur = (double *)malloc(sizeof(double) * (size_t)pop * G);
    double *nxt = (double *)malloc(sizeof(double) * (size_t)pop * G);
    double *fit = (double *)malloc(sizeof(double) * (size_t)pop);
    double *e64 = (double *)malloc(sizeof(double) * (size_t)pop);
    double *a64 = (double *)malloc(sizeof(double) * (size_t)pop);
    float *tot = (float *)malloc(sizeof(float) * (size_t)pop);
    float *xyz = (float *)malloc(sizeof(float) * 3 * (size_t)(n > 0 ? n : 1));
    or_init_population(P, T, seed, lig_index, cur);
    int have = 0;
    float bt = INFINITY;
    int64_t evals = 0;
    for (int gen = 0; gen <= P->generations; ++gen) {
        for (int i = 0; i < pop; ++i) {
            or_pose_into(L, cur + (size_t)i * G, xyz, xyz + n, xyz + 2 * n);
            e64[i] = or_inter_one(L, xyz, xyz + n, xyz + 2 * n);
            a64[i] = L->n_pairs ? or_intra_one(L, xyz, xyz + n, xyz + 2 * n) : 0.0;
            tot[i] = or_total32(e64[i], a64[i], tors32);
            fit[i] = (double)tot[i];
        }
        evals += pop;
        int idx = 0;
        for (int i = 1; i < pop; ++i)
            if (tot[i] < tot[idx]) idx = i;
        if (!have || tot[idx] < bt) {
            have = 1;
            bt = tot[idx];
            memcpy(best_genes, cur + (size_t)idx * G, G * sizeof(double));
            *best_inter = e64[idx];
            *best_intra = a64[idx];
        }
        if (trace) trace[gen] = tot[idx];
        if (gen < P->generations) {
            or_next_generation(P, T, cur, fit, gen, seed, lig_index, nxt, NULL);
            double *s = cur; cur = nxt; nxt = s;
        }
    }
    *best_total = bt;
    *n_evals = evals;
    free(cur); free(nxt); free(fit); free(e64); free(a64); free(tot); free(xyz);
    return 0;
}

/* Many ligands, one OpenMP thread per ligand (the screening CPU baseline). */
int or_dock_many(const or_ligand *ligs, int n_ligs, const or_ga_params *P, uint64_t seed,
                 int64_t lig_index_base, const float *tors32, int g_stride,
                 double *best_genes, float *best_total, double *best_inter,
                 double *best_intra, int64_t *n_evals, int n_threads)
{
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
    for (int l = 0; l < n_ligs; ++l)
        or_dock(&ligs[l], P, seed, (uint64_t)(lig_index_base + l), tors32[l],
                best_genes + (size_t)l * g_stride, &best_total[l], &best_inter[l],
                &best_intra[l], NULL, &n_evals[l]);
    return 0;
}

/* Raw Philox blocks for pinning against numpy. */
void or_philox_block(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                     uint64_t k1, uint64_t *out)
{
    const uint64_t ctr[4] = {c0, c1, c2, c3}, key[2] = {k0, k1};
    or_philox(ctr, key, out);
}

double or_log(double x) { return or_rng_ln(x); }
double or_cos2pi(double u) { return or_rng_cos_2pi(u); }
/* normal of block (c0 = component, c1 = individual, c2 = generation, c3 = phase) */
double or_normal(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0, uint64_t k1)
{
    const or_rng_key key = {k0, k1};
    return or_rng_normal(&key, (int)c3, (int64_t)c2, (int64_t)c1, (int64_t)c0);
}
