/*
 * vd_host.cpp -- batched host preprocessing and the
 * synthetic ligand batches of SURVEY Appendix B, in C++ with OpenMP across
 * ligands.
 *
 * vd_prepare_*  restate, per ligand, the reference's host prep bit for bit:
 *   bond_separation / build_nonbond_pairlist   vd/model.py:195-269
 *   build_fragment_masks                        vd/model.py:174-192
 *   LigandTopology.centroid0 (numpy pairwise mean, fp64 -> f32)  vd/model.py:100-103
 *   _fold_pairs + prepare_context               vd/scoring/__init__.py:117-207
 * producing the vd_ligand_arrays CSR that vd_ligands_create uploads.  The
 * Python path costs 1.4-5.5 ms per ligand; 100k ligands
 * would otherwise take minutes of host time per screen.
 *
 * vd_synth_ligands generates the cfg2/3/4 ligand distributions (random heavy
 * tree, ~1.5 A bonds at tetrahedral-ish angles, HD leaves on N/NA/OA/SA,
 * non-terminal heavy-heavy rotatable bonds, charges U(-0.4,0.4) re-centred),
 * keyed per ligand on a counter-based Philox stream so any index range is
 * generated independently and identically on every host.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "vd_rng.h"
#include "vecdock_b200.h"

namespace {

/* numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * PW_BLOCKSIZE 128) for a contiguous float32 row accumulated in float64 */
double pairwise_sum_f32(const float *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;  /* numpy starts from -0.0; identical for any non-empty sum here */
        for (int64_t i = 0; i < n; ++i) res += (double)a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = (double)a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += (double)a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += (double)a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum_f32(a, n2) + pairwise_sum_f32(a + n2, n - n2);
}

struct Ligand {
    int n;
    const float *xyz;      /* (3, n) */
    const int32_t *type;
    const float *charge;
    int nb;
    const int32_t *bonds;  /* (nb, 2) */
    int nt;
    const int32_t *axes;   /* (nt, 2) axis_a, axis_b */
};

std::vector<std::vector<int>> adjacency(const Ligand &L)
{
    std::vector<std::vector<int>> adj(L.n);
    for (int b = 0; b < L.nb; ++b) {
        const int u = L.bonds[2 * b], v = L.bonds[2 * b + 1];
        adj[u].push_back(v);
        adj[v].push_back(u);
    }
    return adj;
}

/* atoms within 3 bonds of every atom -> mask of excluded pairs (row-major i<j) */
void near_mask(const Ligand &L, const std::vector<std::vector<int>> &adj, std::vector<uint8_t> &near)
{
    const int n = L.n;
    near.assign((size_t)n * n, 0);
    std::vector<int> dist(n, -1), q;
    for (int s = 0; s < n; ++s) {
        std::fill(dist.begin(), dist.end(), -1);
        q.clear();
        q.push_back(s);
        dist[s] = 0;
        for (size_t h = 0; h < q.size(); ++h) {
            const int u = q[h];
            near[(size_t)s * n + u] = 1;
            if (dist[u] == 3) continue;
            for (int v : adj[u])
                if (dist[v] < 0) {
                    dist[v] = dist[u] + 1;
                    q.push_back(v);
                }
        }
    }
}

/* atoms reachable from b with edge (a,b) removed; sorted; -1 on ring */
int fragment(const Ligand &L, const std::vector<std::vector<int>> &adj, int a, int b,
             std::vector<int> &out)
{
    std::vector<uint8_t> seen(L.n, 0);
    std::vector<int> q{b};
    seen[b] = 1;
    for (size_t h = 0; h < q.size(); ++h) {
        const int u = q[h];
        for (int v : adj[u]) {
            if ((u == a && v == b) || (u == b && v == a)) continue;
            if (!seen[v]) {
                seen[v] = 1;
                q.push_back(v);
            }
        }
    }
    if (seen[a]) return -1;
    out.clear();
    for (int i = 0; i < L.n; ++i)
        if (seen[i]) out.push_back(i);
    return 0;
}

}  // namespace

extern "C" {

/* Pass 1: pairs and fragment atoms of each ligand ([L] each); returns 0 or -1 (ring bond). */
int vd_prepare_count(int n_ligands, const int32_t *atom_start, const float *xyz,
                     const int32_t *bond_start, const int32_t *bonds, const int32_t *tors_start,
                     const int32_t *axes, int64_t *n_pairs, int64_t *n_frag)
{
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (int l = 0; l < n_ligands; ++l) {
        Ligand L{atom_start[l + 1] - atom_start[l], nullptr, nullptr, nullptr,
                 bond_start[l + 1] - bond_start[l], bonds + 2 * (int64_t)bond_start[l],
                 tors_start[l + 1] - tors_start[l], axes + 2 * (int64_t)tors_start[l]};
        (void)xyz;
        auto adj = adjacency(L);
        std::vector<uint8_t> near;
        near_mask(L, adj, near);
        int64_t p = 0;
        for (int i = 0; i < L.n; ++i)
            for (int j = i + 1; j < L.n; ++j) p += !near[(size_t)i * L.n + j];
        n_pairs[l] = p;
        int64_t f = 0;
        std::vector<int> frag;
        for (int t = 0; t < L.nt; ++t) {
            if (fragment(L, adj, L.axes[2 * t], L.axes[2 * t + 1], frag)) bad = 1;
            f += (int64_t)frag.size();
        }
        n_frag[l] = f;
    }
    return bad ? -1 : 0;
}

/* Pass 2: fill the ScoringContext CSR (vd_ligand_arrays field order) for every ligand.
 * type_map[type] = grid map index of that type's map (-1: missing -> error). */
int vd_prepare_fill(int n_ligands, const int32_t *atom_start, const float *xyz /* per ligand (3,n) */,
                    const int32_t *type_index, const float *charge, const int32_t *bond_start,
                    const int32_t *bonds, const int32_t *tors_start, const int32_t *axes,
                    const vd_atom_type *table, int n_types, const int32_t *type_map,
                    const vd_weights *w, double w_tors, const int64_t *pair_start,
                    const int64_t *frag_start,
                    /* outputs */
                    float *centered0 /* [sumN][3] */, float *dsf, int32_t *atom_map,
                    int32_t *pair_i, int32_t *pair_j, float *pair_a, float *pair_b,
                    float *pair_qq, float *pair_dsl, uint8_t *pair_hb, int32_t *frag_lo,
                    int32_t *frag_hi, int32_t *frag_index, float *torsional32)
{
    const double QASP = 0.01097, ELEC = 332.06363;
    const float wv = (float)w->vdw, wh = (float)w->hbond;
    const float cq = (float)(w->elec * ELEC), cd = (float)w->desolv;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (int l = 0; l < n_ligands; ++l) {
        const int a0 = atom_start[l];
        Ligand L{atom_start[l + 1] - a0, xyz + 3 * (int64_t)a0, type_index + a0, charge + a0,
                 bond_start[l + 1] - bond_start[l], bonds + 2 * (int64_t)bond_start[l],
                 tors_start[l + 1] - tors_start[l], axes + 2 * (int64_t)tors_start[l]};
        const int n = L.n;
        for (int i = 0; i < n; ++i)
            if (L.type[i] < 0 || L.type[i] >= n_types || type_map[L.type[i]] < 0) bad = 1;
        if (bad) continue;
        /* centroid0 = f32(numpy mean in fp64) ; centred coords in f32 */
        for (int k = 0; k < 3; ++k) {
            const float c = (float)(pairwise_sum_f32(L.xyz + (int64_t)k * n, n) / (double)n);
            for (int i = 0; i < n; ++i) centered0[3 * (int64_t)(a0 + i) + k] = L.xyz[(int64_t)k * n + i] - c;
        }
        for (int i = 0; i < n; ++i) {
            const vd_atom_type &tp = table[L.type[i]];
            dsf[a0 + i] = (float)tp.solpar + (float)QASP * std::fabs(L.charge[i]);
            atom_map[a0 + i] = type_map[L.type[i]];
        }
        auto adj = adjacency(L);
        std::vector<uint8_t> near;
        near_mask(L, adj, near);
        int64_t k = pair_start[l];
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                if (near[(size_t)i * n + j]) continue;
                const vd_atom_type &ti = table[L.type[i]], &tj = table[L.type[j]];
                const double r_eq = 0.5 * (ti.r_eq + tj.r_eq);
                const double eps = std::sqrt(ti.eps * tj.eps);
                const bool hb = (ti.donor && tj.acceptor) || (ti.acceptor && tj.donor);
                const double a = hb ? 5.0 * eps * std::pow(r_eq, 12.0) : eps * std::pow(r_eq, 12.0);
                const double b = hb ? 6.0 * eps * std::pow(r_eq, 10.0) : 2.0 * eps * std::pow(r_eq, 6.0);
                const double qi = (double)L.charge[i], qj = (double)L.charge[j];
                const double d = ti.solpar * tj.volume + tj.solpar * ti.volume +
                                 QASP * (std::fabs(qi) * tj.volume + std::fabs(qj) * ti.volume);
                const float wf = hb ? wh : wv;
                pair_i[k] = i;
                pair_j[k] = j;
                pair_a[k] = wf * (float)a;
                pair_b[k] = wf * (float)b;
                pair_hb[k] = hb;
                pair_qq[k] = cq * (float)(qi * qj);
                pair_dsl[k] = cd * (float)d;
                ++k;
            }
        int64_t f = frag_start[l];
        std::vector<int> frag;
        const int t0 = tors_start[l];
        for (int t = 0; t < L.nt; ++t) {
            if (fragment(L, adj, L.axes[2 * t], L.axes[2 * t + 1], frag)) {
                bad = 1;
                break;
            }
            frag_lo[t0 + t] = (int32_t)f;
            for (int a : frag) frag_index[f++] = a;
            frag_hi[t0 + t] = (int32_t)f;
        }
        torsional32[l] = (float)(w_tors * (double)L.nt);
    }
    return bad ? -1 : 0;
}

/* ---- synthetic ligand batches (cfg2/3/4 recipes) -------------- */
struct Stream {
    uint64_t k0, k1, ctr = 0;
    uint64_t buf[4];
    int pos = 4;
    uint64_t next()
    {
        if (pos == 4) {
            vd_u64x4 w = vd_philox4x64_10(ctr++, 0, 0, 7, k0, k1);
            std::memcpy(buf, w.v, sizeof buf);
            pos = 0;
        }
        return buf[pos++];
    }
    double u01() { return vd_u01(next()); }
    int below(int n) { return (int)vd_below(next(), (uint64_t)n); }
    double normal()
    {
        const double u1 = ((next() >> 11) + 1) * (1.0 / 9007199254740992.0);
        const double u2 = u01();
        return std::sqrt(-2.0 * vd_log(u1)) * vd_cos2pi(u2);
    }
};

/* Sizes of ligand i: heavy ~ U{h_lo..h_hi}, HD = round(heavy * hd_ratio), T ~ U{t_lo..t_hi}. */
static void synth_sizes(uint64_t seed, int64_t i, int h_lo, int h_hi, double hd_ratio, int t_lo,
                        int t_hi, int *heavy, int *hd, int *tors)
{
    Stream s{seed, (uint64_t)i};
    *heavy = h_lo + s.below(h_hi - h_lo + 1);
    *hd = (int)std::lround(*heavy * hd_ratio);
    *tors = t_lo + s.below(t_hi - t_lo + 1);
}

/* type labels used: C A N NA OA SA HD by table index passed in heavy_types[6], hd_type */
int vd_synth_count(uint64_t seed, int64_t first, int count, int h_lo, int h_hi, double hd_ratio,
                   int t_lo, int t_hi, int32_t *n_atoms, int32_t *n_tors_max)
{
    for (int l = 0; l < count; ++l) {
        int h, d, t;
        synth_sizes(seed, first + l, h_lo, h_hi, hd_ratio, t_lo, t_hi, &h, &d, &t);
        n_atoms[l] = h + d;
        n_tors_max[l] = t;
    }
    return 0;
}

int vd_synth_fill(uint64_t seed, int64_t first, int count, int h_lo, int h_hi, double hd_ratio,
                  int t_lo, int t_hi, const int32_t *heavy_types /* [6] */, int32_t hd_type,
                  const int32_t *atom_start, float *xyz /* per ligand (3,n) */, int32_t *type_index,
                  float *charge, int32_t *bonds /* (n-1)*2 per ligand, at 2*(atom_start[l]-l) */,
                  int32_t *n_tors /* [count] actual */, int32_t *axes /* 2*t_hi per ligand */)
{
    const double TETRA = 109.5 * M_PI / 180.0;
#pragma omp parallel for schedule(dynamic, 8)
    for (int l = 0; l < count; ++l) {
        int nh, nd, nt;
        synth_sizes(seed, first + l, h_lo, h_hi, hd_ratio, t_lo, t_hi, &nh, &nd, &nt);
        Stream s{seed, (uint64_t)(first + l)};
        s.ctr = 1ull << 40;  /* disjoint from the size draws */
        const int n = nh + nd, a0 = atom_start[l];
        std::vector<int> parent(n, -1), kids(n, 0), type(n);
        const int backbone = std::min(nh, std::max(nt + 2, (3 * nh) / 5));
        for (int k = 1; k < nh; ++k) {
            if (k < backbone) {
                parent[k] = k - 1;
            } else {
                std::vector<int> open;
                for (int a = 0; a < k; ++a)
                    if (kids[a] < 3) open.push_back(a);
                parent[k] = open[s.below((int)open.size())];
            }
            ++kids[parent[k]];
        }
        for (int k = 0; k < nh; ++k) type[k] = s.below(6);
        for (int h = 0; h < nd; ++h) {  /* HD on N/NA/OA/SA (slots 2..5) with free valence */
            std::vector<int> cand;
            for (int a = 0; a < nh; ++a)
                if (type[a] >= 2 && kids[a] < 3) cand.push_back(a);
            if (cand.empty()) {
                std::vector<int> spare;
                for (int a = 0; a < nh; ++a)
                    if (kids[a] < 3) spare.push_back(a);
                if (spare.empty()) break;
                const int a = spare[s.below((int)spare.size())];
                type[a] = 2 + s.below(4);
                cand.push_back(a);
            }
            const int a = cand[s.below((int)cand.size())];
            parent[nh + h] = a;
            ++kids[a];
        }
        /* geometry */
        std::vector<double> P(3 * (size_t)n, 0.0);
        for (int k = 1; k < n; ++k) {
            const int p = parent[k], g = p >= 0 ? parent[p] : -1;
            const double len = k < nh ? 1.5 + 0.05 * std::max(-2.0, std::min(2.0, s.normal()))
                                      : 1.0 + 0.1 * s.u01();
            double best[3] = {0, 0, 0}, best_c = -1.0;
            for (int tr = 0; tr < 24; ++tr) {
                double d[3];
                if (g < 0) {
                    double x = s.normal(), y = s.normal(), z = s.normal();
                    const double nn = std::sqrt(x * x + y * y + z * z) + 1e-300;
                    d[0] = x / nn; d[1] = y / nn; d[2] = z / nn;
                } else {
                    double b[3] = {P[3 * p] - P[3 * g], P[3 * p + 1] - P[3 * g + 1], P[3 * p + 2] - P[3 * g + 2]};
                    const double bn = std::sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
                    for (double &v : b) v /= bn;
                    double ref[3] = {1, 0, 0};
                    if (std::fabs(b[0]) >= 0.9) { ref[0] = 0; ref[1] = 1; }
                    double e1[3] = {b[1] * ref[2] - b[2] * ref[1], b[2] * ref[0] - b[0] * ref[2], b[0] * ref[1] - b[1] * ref[0]};
                    const double en = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
                    for (double &v : e1) v /= en;
                    const double e2[3] = {b[1] * e1[2] - b[2] * e1[1], b[2] * e1[0] - b[0] * e1[2], b[0] * e1[1] - b[1] * e1[0]};
                    const double ang = TETRA + (s.u01() * 16.0 - 8.0) * M_PI / 180.0;
                    const double phi = 2.0 * M_PI * s.u01();
                    for (int c = 0; c < 3; ++c)
                        d[c] = -std::cos(ang) * b[c] + std::sin(ang) * (std::cos(phi) * e1[c] + std::sin(phi) * e2[c]);
                }
                double c3[3] = {P[3 * p] + len * d[0], P[3 * p + 1] + len * d[1], P[3 * p + 2] + len * d[2]};
                double clr = 1e30;
                for (int q = 0; q < k; ++q) {
                    if (q == p) continue;
                    const double dx = c3[0] - P[3 * q], dy = c3[1] - P[3 * q + 1], dz = c3[2] - P[3 * q + 2];
                    clr = std::min(clr, std::sqrt(dx * dx + dy * dy + dz * dz));
                }
                if (clr > best_c) {
                    best_c = clr;
                    std::memcpy(best, c3, sizeof best);
                }
                if (clr >= 2.0) break;
            }
            std::memcpy(&P[3 * k], best, sizeof best);
        }
        /* charges U(-0.4, 0.4) re-centred to net zero */
        std::vector<double> q(n);
        double qs = 0.0;
        for (int i = 0; i < n; ++i) {
            q[i] = -0.4 + 0.8 * s.u01();
            qs += q[i];
        }
        for (int i = 0; i < n; ++i) {
            charge[a0 + i] = (float)(q[i] - qs / n);
            for (int c = 0; c < 3; ++c) xyz[3 * (int64_t)a0 + (int64_t)c * n + i] = (float)P[3 * i + c];
            type_index[a0 + i] = i < nh ? heavy_types[type[i]] : hd_type;
        }
        int32_t *bl = bonds + 2 * (int64_t)(a0 - l);
        for (int k = 1; k < n; ++k) {
            bl[2 * (k - 1)] = std::min(parent[k], k);
            bl[2 * (k - 1) + 1] = std::max(parent[k], k);
        }
        /* rotatable: non-terminal heavy-heavy tree edges, root-outward, breadth order */
        std::vector<int> hdeg(nh, 0), depth(n, 0), elig;
        for (int k = 1; k < nh; ++k) { ++hdeg[k]; ++hdeg[parent[k]]; }
        for (int k = 1; k < n; ++k) depth[k] = depth[parent[k]] + 1;
        for (int k = 1; k < nh; ++k)
            if (hdeg[k] >= 2 && hdeg[parent[k]] >= 2) elig.push_back(k);
        const int t = std::min(nt, (int)elig.size());
        for (int i = 0; i < t; ++i) {  /* partial Fisher-Yates */
            const int j = i + s.below((int)elig.size() - i);
            std::swap(elig[i], elig[j]);
        }
        std::vector<int> ch(elig.begin(), elig.begin() + t);
        std::sort(ch.begin(), ch.end(), [&](int x, int y) {
            return depth[x] != depth[y] ? depth[x] < depth[y] : x < y;
        });
        n_tors[l] = t;
        int32_t *ax = axes + 2 * (int64_t)t_hi * l;
        for (int i = 0; i < t; ++i) {
            ax[2 * i] = parent[ch[i]];
            ax[2 * i + 1] = ch[i];
        }
    }
    return 0;
}

}  // extern "C"
