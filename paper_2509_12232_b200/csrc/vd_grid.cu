/*
 * vd_grid.cu -- AutoGrid-style receptor map builder on the device.
 *
 * Restates vd/grids.py:122-202 (build_grid_maps): per node, an fp64 sum over
 * receptor atoms IN RECEPTOR ORDER (the order numpy accumulates in), elec
 * without cutoff, vdW/H-bond/desolvation within `cutoff`, weights folded.
 * One thread per node (z fastest -> coalesced map writes); receptor atoms are
 * staged through shared memory in tiles so every thread of the CTA reads the
 * same atom at the same time (broadcast).  The per-(probe, receptor type)
 * well coefficients are computed on the host with the reference's fp64
 * expressions and passed in.  fp64 throughout: near receptor atoms map
 * values reach ~5e17 and the maps are parity-checked at rel 1e-4
 * (pkg/tests/test_grids.py:97-118).
 */
#include <cmath>
#include <vector>

#include "vd_internal.h"

namespace vd {

constexpr int kGridTile = 256;
constexpr int kMaxProbe = 16;
constexpr int kMaxTypes = 32;

struct GridBuildArgs {
    const float *rx, *ry, *rz, *rq;
    const int *rt;
    int n_rec;
    int n_probe, n_types;
    const double *c_a, *c_b;   /* [n_probe][n_types] */
    const int *c_hb;
    const double *probe_vol;   /* [n_probe] w_desolv * volume(probe) */
    const double *rec_vol;     /* [n_types] w_desolv * volume(type) */
    const double *rec_sol;     /* [n_types] solpar(type) */
    double ox, oy, oz, spacing;
    int nx, ny, nz;
    double w_vdw, w_hb, elec_pref, cutoff2;
    float *out;
};

__global__ void __launch_bounds__(kGridTile) grid_kernel(GridBuildArgs a)
{
    __shared__ double sx[kGridTile], sy[kGridTile], sz[kGridTile], sq[kGridTile];
    __shared__ int st[kGridTile];
    __shared__ double s_ca[kMaxProbe * kMaxTypes], s_cb[kMaxProbe * kMaxTypes];
    __shared__ int s_hb[kMaxProbe * kMaxTypes];
    const int nt = a.n_probe * a.n_types;
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
        s_ca[k] = a.c_a[k];
        s_cb[k] = a.c_b[k];
        s_hb[k] = a.c_hb[k];
    }
    const int64_t n_nodes = (int64_t)a.nx * a.ny * a.nz;
    const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = node < n_nodes;
    const int iz = (int)(node % a.nz), iy = (int)((node / a.nz) % a.ny),
              ix = (int)(node / ((int64_t)a.ny * a.nz));
    const double gx = __dadd_rn(a.ox, __dmul_rn(a.spacing, (double)ix));
    const double gy = __dadd_rn(a.oy, __dmul_rn(a.spacing, (double)iy));
    const double gz = __dadd_rn(a.oz, __dmul_rn(a.spacing, (double)iz));
    double acc[kMaxProbe];
#pragma unroll
    for (int t = 0; t < kMaxProbe; ++t) acc[t] = 0.0;
    double elec = 0.0, desolv = 0.0;
    const double DB = 78.4 - -8.5525;
    const double lam = -0.003627 * DB;
    for (int base = 0; base < a.n_rec; base += kGridTile) {
        __syncthreads();
        const int j = base + threadIdx.x;
        if (j < a.n_rec) {
            sx[threadIdx.x] = (double)a.rx[j];
            sy[threadIdx.x] = (double)a.ry[j];
            sz[threadIdx.x] = (double)a.rz[j];
            sq[threadIdx.x] = (double)a.rq[j];
            st[threadIdx.x] = a.rt[j];
        }
        __syncthreads();
        const int cnt = min(kGridTile, a.n_rec - base);
        if (!live) continue;
        for (int u = 0; u < cnt; ++u) {
            const double dx = __dsub_rn(gx, sx[u]), dy = __dsub_rn(gy, sy[u]),
                         dz = __dsub_rn(gz, sz[u]);
            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            const double r = __dsqrt_rn(r2);
            const double rc = r > 0.1 ? r : 0.1;
            const double eps_r = __dadd_rn(-8.5525, __ddiv_rn(DB, __dadd_rn(1.0, __dmul_rn(7.7839, exp(__dmul_rn(lam, rc))))));
            elec = __dadd_rn(elec, __ddiv_rn(__dmul_rn(a.elec_pref, sq[u]), __dmul_rn(rc, eps_r)));
            if (!(r2 <= a.cutoff2)) continue;
            const int ty = st[u];
            const double gauss = exp(__ddiv_rn(-r2, 2.0 * 3.6 * 3.6));
            desolv = __dadd_rn(desolv, __dmul_rn(a.rec_vol[ty], gauss));
            const double sj = __dadd_rn(a.rec_sol[ty], __dmul_rn(0.01097, fabs(sq[u])));
            const double r2c = r2 > 0.01 ? r2 : 0.01;
            const double inv = __ddiv_rn(1.0, r2c);
            const double i2 = __dmul_rn(inv, inv);
            const double i3 = __dmul_rn(i2, inv);
            const double i6 = __dmul_rn(i3, i3);
            for (int t = 0; t < a.n_probe; ++t) {
                const int k = t * a.n_types + ty;
                double well;
                if (s_hb[k])
                    well = __dmul_rn(a.w_hb, __dsub_rn(__dmul_rn(s_ca[k], i6), __dmul_rn(s_cb[k], __dmul_rn(i3, i2))));
                else
                    well = __dmul_rn(a.w_vdw, __dsub_rn(__dmul_rn(s_ca[k], i6), __dmul_rn(s_cb[k], i3)));
                const double pd = __dmul_rn(__dmul_rn(a.probe_vol[t], sj), gauss);
                acc[t] = __dadd_rn(acc[t], __dadd_rn(well, pd));
            }
        }
    }
    if (!live) return;
#pragma unroll
    for (int t = 0; t < kMaxProbe; ++t)
        if (t < a.n_probe) a.out[t * n_nodes + node] = __double2float_rn(acc[t]);
    a.out[(int64_t)a.n_probe * n_nodes + node] = __double2float_rn(elec);
    a.out[(int64_t)(a.n_probe + 1) * n_nodes + node] = __double2float_rn(desolv);
}

}  // namespace vd

using vdi::set_error;

extern "C" int vd_grid_build(const float *rec_xyz, const int32_t *rec_type, const float *rec_charge,
                             int n_rec, const vd_atom_type *table, int n_types,
                             const int32_t *probe, int n_probe, const double origin[3],
                             double spacing, int nx, int ny, int nz, const vd_weights *w,
                             double cutoff, vd_grid **out)
{
    *out = nullptr;
    if (n_probe < 1 || n_probe > vd::kMaxProbe || n_types < 1 || n_types > vd::kMaxTypes ||
        n_rec < 1) {
        set_error("vd_grid_build: need 1..16 probe types, 1..32 table types, >= 1 receptor atom");
        return -1;
    }
    for (int j = 0; j < n_rec; ++j)
        if (rec_type[j] < 0 || rec_type[j] >= n_types) {
            set_error("vd_grid_build: receptor atom type index out of range");
            return -1;
        }
    /* host-side coefficient tables with the reference's Python-float arithmetic */
    std::vector<double> ca(n_probe * n_types), cb(n_probe * n_types), pv(n_probe), rv(n_types),
        rs(n_types);
    std::vector<int> hb(n_probe * n_types);
    for (int t = 0; t < n_probe; ++t) {
        const vd_atom_type &pt = table[probe[t]];
        pv[t] = (w->desolv * pt.volume);
        for (int r = 0; r < n_types; ++r) {
            const vd_atom_type &pr = table[r];
            const double r_eq = 0.5 * (pt.r_eq + pr.r_eq);
            const double eps = std::sqrt(pt.eps * pr.eps);
            const int h = (pt.donor && pr.acceptor) || (pt.acceptor && pr.donor);
            const int k = t * n_types + r;
            hb[k] = h;
            if (h) { ca[k] = 5.0 * eps * std::pow(r_eq, 12.0); cb[k] = 6.0 * eps * std::pow(r_eq, 10.0); }
            else { ca[k] = eps * std::pow(r_eq, 12.0); cb[k] = 2.0 * eps * std::pow(r_eq, 6.0); }
        }
    }
    for (int r = 0; r < n_types; ++r) {
        rv[r] = w->desolv * table[r].volume;
        rs[r] = table[r].solpar;
    }
    vd_grid *g = nullptr;
    const float lo[3] = {(float)origin[0], (float)origin[1], (float)origin[2]};
    const float hi[3] = {(float)(origin[0] + (nx - 1) * spacing), (float)(origin[1] + (ny - 1) * spacing),
                         (float)(origin[2] + (nz - 1) * spacing)};
    if (vd_grid_create(nullptr, n_probe + 2, nx, ny, nz, lo, hi, (float)spacing, &g)) return -1;
    float *d_rec = nullptr;
    int *d_rt = nullptr;
    double *d_tab = nullptr;
    int *d_hb = nullptr;
    const size_t ntab = ca.size() * 2 + pv.size() + rv.size() + rs.size();
    std::vector<double> tab;
    tab.insert(tab.end(), ca.begin(), ca.end());
    tab.insert(tab.end(), cb.begin(), cb.end());
    tab.insert(tab.end(), pv.begin(), pv.end());
    tab.insert(tab.end(), rv.begin(), rv.end());
    tab.insert(tab.end(), rs.begin(), rs.end());
    bool ok = vdi::check(cudaMalloc(&d_rec, sizeof(float) * 4 * n_rec), "alloc rec") &&
              vdi::check(cudaMalloc(&d_rt, sizeof(int) * n_rec), "alloc rt") &&
              vdi::check(cudaMalloc(&d_tab, sizeof(double) * ntab), "alloc tab") &&
              vdi::check(cudaMalloc(&d_hb, sizeof(int) * hb.size()), "alloc hb") &&
              vdi::check(cudaMemcpy(d_rec, rec_xyz, sizeof(float) * 3 * n_rec, cudaMemcpyDefault), "up xyz") &&
              vdi::check(cudaMemcpy(d_rec + 3 * n_rec, rec_charge, sizeof(float) * n_rec, cudaMemcpyDefault), "up q") &&
              vdi::check(cudaMemcpy(d_rt, rec_type, sizeof(int) * n_rec, cudaMemcpyDefault), "up t") &&
              vdi::check(cudaMemcpy(d_tab, tab.data(), sizeof(double) * ntab, cudaMemcpyHostToDevice), "up tab") &&
              vdi::check(cudaMemcpy(d_hb, hb.data(), sizeof(int) * hb.size(), cudaMemcpyHostToDevice), "up hb");
    if (ok) {
        vd::GridBuildArgs a;
        a.rx = d_rec; a.ry = d_rec + n_rec; a.rz = d_rec + 2 * n_rec; a.rq = d_rec + 3 * n_rec;
        a.rt = d_rt;
        a.n_rec = n_rec;
        a.n_probe = n_probe;
        a.n_types = n_types;
        a.c_a = d_tab;
        a.c_b = d_tab + ca.size();
        a.probe_vol = d_tab + 2 * ca.size();
        a.rec_vol = a.probe_vol + n_probe;
        a.rec_sol = a.rec_vol + n_types;
        a.c_hb = d_hb;
        a.ox = origin[0]; a.oy = origin[1]; a.oz = origin[2];
        a.spacing = spacing;
        a.nx = nx; a.ny = ny; a.nz = nz;
        a.w_vdw = w->vdw;
        a.w_hb = w->hbond;
        a.elec_pref = w->elec * 332.06363;
        a.cutoff2 = cutoff * cutoff;
        a.out = g->d_maps;
        const int64_t n_nodes = (int64_t)nx * ny * nz;
        vd::grid_kernel<<<(unsigned)((n_nodes + vd::kGridTile - 1) / vd::kGridTile), vd::kGridTile>>>(a);
        ++vdi::g_launches;
        ok = vdi::check(cudaGetLastError(), "grid kernel") &&
             vdi::check(cudaDeviceSynchronize(), "grid kernel sync") && vdi::make_packed(g);
    }
    cudaFree(d_rec);
    cudaFree(d_rt);
    cudaFree(d_tab);
    cudaFree(d_hb);
    if (!ok) {
        vd_grid_destroy(g);
        return -1;
    }
    *out = g;
    return 0;
}
