/*
 * vd_oracle.c -- CPU restatement of the reference's docking hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU baseline timed by bench.py (`cpu_baseline`,
 * `--impl reference`).  Only tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs load it; the product package never does.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * fixtures produced by the reference itself (tests/golden/make_golden.py,
 * which imports /root/reference/pkg/src/vecdock), bit-for-bit on inter64 /
 * intra64 / total32 and poses, and against the reference's own golden vector
 * pkg/tests/data/golden_score.json at its 1e-4 tolerance.
 *
 * Build: oracle/Makefile (-O2 -ffp-contract=off: the reference's float32 and
 * float64 sequences contain no fused multiply-adds, and glibc supplies the
 * same exp/cos/sin/sqrt that numba's nopython code calls).
 *
 * Sequences restated (file:line under /root/reference/pkg/src/vecdock):
 *   pose      scoring/simd.py:157-222  (== pose.py:137-205)
 *   inter     scoring/simd.py:89-138   (== scoring/reference.py:73-84,113-148)
 *   intra     scoring/simd.py:36-86    (== scoring/reference.py:52-70,87-111)
 *   totals    scoring/__init__.py:330-346 (f32(f32(inter)+f32(intra)) + tors32)
 *   grid      grids.py:122-202 (fp64 direct sum, receptor order per node)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- constants: energy.py:17-34, scoring/__init__.py:42 ---------------- */
static const double ELEC_SCALE = 332.06363;
static const double DIEL_A = -8.5525;
#define DIEL_B_EXPR (78.4 - -8.5525)
static const double DIEL_K = 7.7839;
static const double DIEL_LAMBDA = 0.003627;
#define DESOLV_DENOM_EXPR (2.0 * 3.6 * 3.6)
static const double QASP = 0.01097;
static const float MIN_R2F = 0.01f;
static const double MIN_R2 = 0.01;
static const double MIN_R = 0.1;

#include "vd_oracle.h"

/* --- A1: pose (simd.py:157-222) ----------------------------------------- */
void or_pose_into(const or_ligand *L, const double *g, float *px, float *py, float *pz)
{
    const int n = L->n_atoms;
    double q0 = g[3], q1 = g[4], q2 = g[5], q3 = g[6];
    double norm = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    double w = q0 / norm, x = q1 / norm, y = q2 / norm, z = q3 / norm;
    float m00 = (float)(1.0 - 2.0 * (y * y + z * z));
    float m01 = (float)(2.0 * (x * y - w * z));
    float m02 = (float)(2.0 * (x * z + w * y));
    float m10 = (float)(2.0 * (x * y + w * z));
    float m11 = (float)(1.0 - 2.0 * (x * x + z * z));
    float m12 = (float)(2.0 * (y * z - w * x));
    float m20 = (float)(2.0 * (x * z - w * y));
    float m21 = (float)(2.0 * (y * z + w * x));
    float m22 = (float)(1.0 - 2.0 * (x * x + y * y));
    float tx = (float)g[0], ty = (float)g[1], tz = (float)g[2];
    const float *cx = L->centered0, *cy = cx + n, *cz = cx + 2 * n;
    for (int i = 0; i < n; ++i) {
        px[i] = ((m00 * cx[i] + m01 * cy[i]) + m02 * cz[i]) + tx;
        py[i] = ((m10 * cx[i] + m11 * cy[i]) + m12 * cz[i]) + ty;
        pz[i] = ((m20 * cx[i] + m21 * cy[i]) + m22 * cz[i]) + tz;
    }
    for (int t = 0; t < L->n_torsions; ++t) {
        int ia = L->axis_a[t], ib = L->axis_b[t];
        float ox = px[ia], oy = py[ia], oz = pz[ia];
        double ax = (double)(px[ib] - ox), ay = (double)(py[ib] - oy), az = (double)(pz[ib] - oz);
        double an = sqrt((ax * ax + ay * ay) + az * az);
        float kx = (float)(ax / an), ky = (float)(ay / an), kz = (float)(az / an);
        double th = g[7 + t];
        float c = (float)cos(th), s = (float)sin(th);
        float omc = 1.0f - c;
        for (int f = L->frag_start[t]; f < L->frag_start[t + 1]; ++f) {
            int i = L->frag_index[f];
            float vx = px[i] - ox, vy = py[i] - oy, vz = pz[i] - oz;
            float dot = (kx * vx + ky * vy) + kz * vz;
            float cxx = ky * vz - kz * vy;
            float cxy = kz * vx - kx * vz;
            float cxz = kx * vy - ky * vx;
            px[i] = ((vx * c + cxx * s) + kx * (dot * omc)) + ox;
            py[i] = ((vy * c + cxy * s) + ky * (dot * omc)) + oy;
            pz[i] = ((vz * c + cxz * s) + kz * (dot * omc)) + oz;
        }
    }
}

/* --- A2: inter (simd.py:89-138) ------------------------------------------ */
static inline float lerpf_(float a, float b, float t) { return a * (1.0f - t) + b * t; }

static float trilerp(const float *m, int ny, int nz, int ix, int iy, int iz,
                     float fx, float fy, float fz)
{
#define V(a, b, c) m[((size_t)(ix + (a)) * ny + (iy + (b))) * nz + (iz + (c))]
    float c00 = lerpf_(V(0, 0, 0), V(1, 0, 0), fx);
    float c10 = lerpf_(V(0, 1, 0), V(1, 1, 0), fx);
    float c01 = lerpf_(V(0, 0, 1), V(1, 0, 1), fx);
    float c11 = lerpf_(V(0, 1, 1), V(1, 1, 1), fx);
#undef V
    float c0 = lerpf_(c00, c10, fy);
    float c1 = lerpf_(c01, c11, fy);
    return lerpf_(c0, c1, fz);
}

double or_inter_one(const or_ligand *L, const float *px, const float *py, const float *pz)
{
    const size_t msz = (size_t)L->nx * L->ny * L->nz;
    const float lo0 = L->lo[0], lo1 = L->lo[1], lo2 = L->lo[2];
    const float hi0 = L->hi[0], hi1 = L->hi[1], hi2 = L->hi[2];
    double acc = 0.0;
    for (int i = 0; i < L->n_atoms; ++i) {
        float x = px[i], y = py[i], z = pz[i], term;
        if (x >= lo0 && x <= hi0 && y >= lo1 && y <= hi1 && z >= lo2 && z <= hi2) {
            float ux = (x - lo0) / L->spacing, uy = (y - lo1) / L->spacing, uz = (z - lo2) / L->spacing;
            int ix = (int)ux, iy = (int)uy, iz = (int)uz;
            if (ix > L->nx - 2) ix = L->nx - 2;
            if (iy > L->ny - 2) iy = L->ny - 2;
            if (iz > L->nz - 2) iz = L->nz - 2;
            float fx = ux - (float)ix, fy = uy - (float)iy, fz = uz - (float)iz;
            float t = trilerp(L->maps + msz * L->atom_map[i], L->ny, L->nz, ix, iy, iz, fx, fy, fz);
            float e = L->charge[i] * trilerp(L->maps + msz * L->elec_map, L->ny, L->nz, ix, iy, iz, fx, fy, fz);
            float d = L->dsf[i] * trilerp(L->maps + msz * L->desolv_map, L->ny, L->nz, ix, iy, iz, fx, fy, fz);
            term = (t + e) + d;
        } else {
            float dx = fmaxf(fmaxf(lo0 - x, x - hi0), 0.0f);
            float dy = fmaxf(fmaxf(lo1 - y, y - hi1), 0.0f);
            float dz = fmaxf(fmaxf(lo2 - z, z - hi2), 0.0f);
            float dist = sqrtf((dx * dx + dy * dy) + dz * dz);
            term = L->penalty * (dist + 1.0f);
        }
        acc += (double)term;
    }
    return acc;
}

/* --- A3: intra (simd.py:36-86) ------------------------------------------- */
static inline float pair_term(float dx, float dy, float dz, float a, float b, int hb,
                              float qq, float dsl, float cut2)
{
    const double DIEL_B = DIEL_B_EXPR;
    const double LAMB = DIEL_LAMBDA * DIEL_B_EXPR;
    float r2 = (dx * dx + dy * dy) + dz * dz;
    if (r2 > cut2) return 0.0f;
    float r2c = r2 > MIN_R2F ? r2 : MIN_R2F;
    float inv = 1.0f / r2c;
    float i2 = inv * inv;
    float i3 = i2 * inv;
    float i6 = i3 * i3;
    float well = hb ? a * i6 - b * (i3 * i2) : a * i6 - b * i3;
    float r = sqrtf(r2c);
    double r64 = (double)r;
    double eps_r = DIEL_A + DIEL_B / (1.0 + DIEL_K * exp(-(LAMB * r64)));
    float elec = (float)((double)qq / (r64 * eps_r));
    float desolv = (float)((double)dsl * exp(-((double)r2 / DESOLV_DENOM_EXPR)));
    return (well + elec) + desolv;
}

double or_intra_one(const or_ligand *L, const float *px, const float *py, const float *pz)
{
    const int n = L->n_pairs, lane = L->lane > 0 ? L->lane : 8;
    double lane_acc[64];
    int nl = lane > 64 ? 64 : lane;
    for (int l = 0; l < nl; ++l) lane_acc[l] = 0.0;
    int nblk = n / nl;
    for (int blk = 0; blk < nblk; ++blk)
        for (int l = 0; l < nl; ++l) {
            int k = blk * nl + l, i = L->pi[k], j = L->pj[k];
            lane_acc[l] += (double)pair_term(px[i] - px[j], py[i] - py[j], pz[i] - pz[j],
                                             L->pa[k], L->pb[k], L->phb[k], L->pqq[k], L->pdsl[k], L->cut2);
        }
    double tail = 0.0;
    for (int k = nblk * nl; k < n; ++k) {
        int i = L->pi[k], j = L->pj[k];
        tail += (double)pair_term(px[i] - px[j], py[i] - py[j], pz[i] - pz[j],
                                  L->pa[k], L->pb[k], L->phb[k], L->pqq[k], L->pdsl[k], L->cut2);
    }
    double total = 0.0;
    for (int l = 0; l < nl; ++l) total += lane_acc[l];
    return total + tail;
}

/* --- population entries (simd.py:141-154, 225-240; __init__.py:330-346) -- */
float or_total32(double inter, double intra, float tors)
{
    float s = (float)inter + (float)intra;
    return s + tors;
}

int or_dock_population(const or_ligand *L, const double *genes, int64_t P, int G,
                       double *inter, double *intra, float *total, float tors32, int n_threads)
{
    const int n = L->n_atoms;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel num_threads(n_threads)
#endif
    {
        float *buf = (float *)malloc(sizeof(float) * 3 * (size_t)(n > 0 ? n : 1));
        float *px = buf, *py = buf + n, *pz = buf + 2 * n;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
        for (int64_t p = 0; p < P; ++p) {
            or_pose_into(L, genes + p * G, px, py, pz);
            double e = or_inter_one(L, px, py, pz);
            double a = L->n_pairs ? or_intra_one(L, px, py, pz) : 0.0;
            inter[p] = e;
            intra[p] = a;
            if (total) total[p] = or_total32(e, a, tors32);
        }
        free(buf);
    }
    return 0;
}

int or_score_poses(const or_ligand *L, const float *poses, int64_t P,
                   double *inter, double *intra, int n_threads)
{
    const int n = L->n_atoms;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(n_threads)
#endif
    for (int64_t p = 0; p < P; ++p) {
        const float *x = poses + (size_t)p * 3 * n;
        inter[p] = or_inter_one(L, x, x + n, x + 2 * n);
        intra[p] = L->n_pairs ? or_intra_one(L, x, x + n, x + 2 * n) : 0.0;
    }
    return 0;
}

int or_pose_population(const or_ligand *L, const double *genes, int64_t P, int G, float *out)
{
    const int n = L->n_atoms;
    for (int64_t p = 0; p < P; ++p) {
        float *x = out + (size_t)p * 3 * n;
        or_pose_into(L, genes + p * G, x, x + n, x + 2 * n);
    }
    return 0;
}

/* --- grid maps (grids.py:122-202) ----------------------------------------- */
typedef struct {
    double r_eq, eps, volume, solpar;
    int donor, acceptor;
} or_atom_type;

int or_build_grid(const float *pcoords /* (3, na) */, const int32_t *ptype, const float *pcharge,
                  int na, const or_atom_type *table, int n_types,
                  const int32_t *probe, int n_probe,
                  double ox, double oy, double oz, double spacing, int nx, int ny, int nz,
                  double w_vdw, double w_hb, double w_elec, double w_desolv, double cutoff,
                  float *out /* (n_probe + 2, nx, ny, nz) */, int n_threads)
{
    (void)n_types;
    const double DIEL_B = DIEL_B_EXPR;
    const double cutoff2 = cutoff * cutoff;
    const size_t msz = (size_t)nx * ny * nz;
    const double elec_pref = w_elec * ELEC_SCALE;           /* (w_e * E) * q_j */
    const double lam = -DIEL_LAMBDA * DIEL_B;                /* (-l * B) * r   */
    /* per (probe, receptor-type) well coefficients, Python-float arithmetic */
    double *c_a = (double *)malloc(sizeof(double) * (size_t)n_probe * n_types);
    double *c_b = (double *)malloc(sizeof(double) * (size_t)n_probe * n_types);
    int *c_hb = (int *)malloc(sizeof(int) * (size_t)n_probe * n_types);
    for (int t = 0; t < n_probe; ++t)
        for (int r = 0; r < n_types; ++r) {
            const or_atom_type *pt = &table[probe[t]], *pr = &table[r];
            double r_eq = 0.5 * (pt->r_eq + pr->r_eq);
            double eps = sqrt(pt->eps * pr->eps);
            int hb = (pt->donor && pr->acceptor) || (pt->acceptor && pr->donor);
            size_t k = (size_t)t * n_types + r;
            c_hb[k] = hb;
            if (hb) { c_a[k] = 5.0 * eps * pow(r_eq, 12.0); c_b[k] = 6.0 * eps * pow(r_eq, 10.0); }
            else { c_a[k] = eps * pow(r_eq, 12.0); c_b[k] = 2.0 * eps * pow(r_eq, 6.0); }
        }
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(n_threads) collapse(2)
#endif
    for (int ix = 0; ix < nx; ++ix)
        for (int iy = 0; iy < ny; ++iy) {
            double acc[64 + 2];
            for (int iz = 0; iz < nz; ++iz) {
                double gx = ox + spacing * (double)ix, gy = oy + spacing * (double)iy,
                       gz = oz + spacing * (double)iz;
                for (int t = 0; t < n_probe + 2; ++t) acc[t] = 0.0;
                for (int j = 0; j < na; ++j) {
                    const or_atom_type *pr = &table[ptype[j]];
                    double qj = (double)pcharge[j];
                    double dx = gx - (double)pcoords[j], dy = gy - (double)pcoords[na + j],
                           dz = gz - (double)pcoords[2 * na + j];
                    double r2 = (dx * dx + dy * dy) + dz * dz;
                    double r = sqrt(r2);
                    double rc = r > MIN_R ? r : MIN_R;
                    double eps_r = DIEL_A + DIEL_B / (1.0 + DIEL_K * exp(lam * rc));
                    acc[n_probe] += (elec_pref * qj) / (rc * eps_r);
                    if (!(r2 <= cutoff2)) continue;
                    double gauss = exp(-r2 / DESOLV_DENOM_EXPR);
                    acc[n_probe + 1] += (w_desolv * pr->volume) * gauss;
                    double sj = pr->solpar + QASP * fabs(qj);
                    double r2c = r2 > MIN_R2 ? r2 : MIN_R2;
                    double inv = 1.0 / r2c;
                    for (int t = 0; t < n_probe; ++t) {
                        size_t k = (size_t)t * n_types + ptype[j];
                        double well;
                        if (c_hb[k]) {
                            double i2 = inv * inv, i3 = i2 * inv;
                            well = w_hb * (c_a[k] * (i3 * i3) - c_b[k] * (i3 * i2));
                        } else {
                            double i3 = (inv * inv) * inv;
                            well = w_vdw * (c_a[k] * (i3 * i3) - c_b[k] * i3);
                        }
                        double pd = ((w_desolv * table[probe[t]].volume) * sj) * gauss;
                        acc[t] += well + pd;
                    }
                }
                size_t node = ((size_t)ix * ny + iy) * nz + iz;
                for (int t = 0; t < n_probe + 2; ++t) out[t * msz + node] = (float)acc[t];
            }
        }
    free(c_a); free(c_b); free(c_hb);
    return 0;
}
