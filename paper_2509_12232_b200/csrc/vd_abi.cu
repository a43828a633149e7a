/*
 * vd_abi.cu -- the extern "C" boundary of libvdb200.so (see include/vecdock_b200.h).
 *
 * Handles own device memory; bulk arguments may be host or device pointers.
 * Host-resident genotype batches are streamed through a two-stream chunk
 * pipeline (H2D copy of chunk c+1 and D2H of chunk c-1 overlap the kernel on
 * chunk c), which is what the e2e bench line measures.
 */
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "vd_internal.h"

/* L2 share a packed copy may touch: B200's 126 MB L2 is split over two dies and lines
 * read from both dies are cached on both, so a map set gathered by every SM thrashes
 * well below 126 MB (cfg1: the 74 MB yz-brick copy read 1.19 GB of DRAM per 1M-pose
 * launch; the 45 MB z-pair copy 166 MB) */
#ifndef VD_BRICK_BUDGET_MB
#define VD_BRICK_BUDGET_MB 48
#endif

namespace vd {
cudaError_t launch_score(int mode, int src, const GridView &G, const LigView &L,
                         const double *genes, const float *poses, int64_t P, int ngenes,
                         double *inter, double *intra, float *total, cudaStream_t st);
cudaError_t launch_pose(const LigView &L, const double *genes, int64_t P, int ngenes, float *out,
                        cudaStream_t st, int tpp_force);
}  // namespace vd

namespace vdi {
static thread_local std::string g_err;
thread_local int64_t g_launches = 0;

void set_error(const std::string &msg) { g_err = msg; }

static thread_local std::string g_detail;  /* why a launch helper refused (set_detail) */

void set_detail(const std::string &msg) { g_detail = msg; }

bool check(cudaError_t e, const char *what)
{
    if (e == cudaSuccess) return true;
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    if (!g_detail.empty()) g_err += " (" + g_detail + ")";
    g_detail.clear();
    cudaGetLastError();
    return false;
}

bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

__global__ void pack_yz(const float *__restrict__ maps, int64_t n, int ny, int nz, float4 *yz)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const bool zl = (k % nz) == nz - 1, yl = ((k / nz) % ny) == ny - 1;
        yz[k] = make_float4(maps[k], zl ? 0.f : maps[k + 1], yl ? 0.f : maps[k + nz],
                            (zl || yl) ? 0.f : maps[k + nz + 1]);
    }
}

/* zy layout: z-pair (v[z], v[z+1]) of node (x, y, z) at ((x*nyp + y/2)*nz + z)*2 + (y&1) */
__global__ void pack_zy(const float *__restrict__ maps, int64_t n, int ny, int nz, float2 *zp)
{
    const int nyp = (ny + 1) / 2;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(k % nz);
        const int64_t xy = k / nz;
        const int y = (int)(xy % ny);
        const int64_t x = xy / ny;
        zp[((x * nyp + (y >> 1)) * nz + z) * 2 + (y & 1)] =
            make_float2(maps[k], z == nz - 1 ? 0.f : maps[k + 1]);
    }
}

__global__ void pack_ed(const float *__restrict__ e, const float *__restrict__ d, int64_t n,
                        int ny, int nz, float4 *ed)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const bool zl = (k % nz) == nz - 1, yl = ((k / nz) % ny) == ny - 1;
        ed[2 * k] = make_float4(e[k], zl ? 0.f : e[k + 1], yl ? 0.f : e[k + nz],
                                (zl || yl) ? 0.f : e[k + nz + 1]);
        ed[2 * k + 1] = make_float4(d[k], zl ? 0.f : d[k + 1], yl ? 0.f : d[k + nz],
                                    (zl || yl) ? 0.f : d[k + nz + 1]);
    }
}

/* Build the packed gather copy when it stays L2-resident.  Type maps are yz-bricks (2
 * LDG.128 per atom) when the touched copy -- every type map plus the 32-B elec/desolv
 * bricks -- fits the budget above, else z-pairs (4 LDG.64 per atom, half the footprint;
 * cfg2's 64^3 grid takes bricks, cfg1's 80^3 z-pairs), else nothing (plain gathers). */
bool make_packed(vd_grid *g)
{
    const int64_t nodes = (int64_t)g->nx * g->ny * g->nz;
    const int64_t n_type = g->n_maps > 2 ? g->n_maps - 2 : 1;
    const int64_t zy_nodes = (int64_t)g->nx * (2 * ((g->ny + 1) / 2)) * g->nz;
    const int64_t brick = nodes * (16 * n_type + 32), zpair = zy_nodes * 8 * n_type + nodes * 32;
    if (getenv("VD_NO_PACK") || zpair > (int64_t)96 << 20) return true;
    const char *ov = getenv("VD_BRICK_BUDGET_MB");  /* tests force either layout */
    g->zpair = brick > ((ov ? atoll(ov) : (int64_t)VD_BRICK_BUDGET_MB) << 20);
    /* type maps are packed lazily in ed_for(): only the maps a ligand set can
       reference (every map except its elec/desolv pair) */
    g->yz_packed.assign(g->n_maps, 0);
    g->tstride = g->zpair ? zy_nodes : nodes;
    if (!check(cudaMalloc(&g->d_yz, (g->zpair ? sizeof(float2) : sizeof(float4)) * g->tstride * g->n_maps), "alloc yz"))
        return false;
    /* zy rows past ny (odd ny) are never read as corners but are gathered as the 2nd
       half of a 16-B group: keep them defined */
    return check(cudaMemset(g->d_yz, 0, (g->zpair ? sizeof(float2) : sizeof(float4)) * g->tstride * g->n_maps), "zero yz");
}

static const float4 *ed_for(const vd_grid *gc, int e, int d)
{
    vd_grid *g = const_cast<vd_grid *>(gc);
    if (!g->d_yz || e < 0 || d < 0 || e >= g->n_maps || d >= g->n_maps) return nullptr;
    std::lock_guard<std::mutex> lk(g->ed_lock);
    auto it = g->d_ed.find({e, d});
    if (it != g->d_ed.end()) return it->second;
    const int64_t nodes = (int64_t)g->nx * g->ny * g->nz;
    float4 *p = nullptr;
    if (cudaMalloc(&p, 2 * sizeof(float4) * nodes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    pack_ed<<<1184, 256>>>(g->d_maps + nodes * e, g->d_maps + nodes * d, nodes, g->ny, g->nz, p);
    for (int m = 0; m < g->n_maps; ++m)
        if (m != e && m != d && !g->yz_packed[m]) {
            if (g->zpair)
                pack_zy<<<1184, 256>>>(g->d_maps + nodes * m, nodes, g->ny, g->nz,
                                       reinterpret_cast<float2 *>(g->d_yz) + g->tstride * m);
            else
                pack_yz<<<1184, 256>>>(g->d_maps + nodes * m, nodes, g->ny, g->nz, g->d_yz + g->tstride * m);
            g->yz_packed[m] = 1;
        }
    if (cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        return nullptr;
    }
    g->d_ed[{e, d}] = p;
    return p;
}

cudaError_t raise_smem_limit(const void *kernel, unsigned bytes)
{
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, unsigned> limits;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    unsigned &cur = limits[{dev, kernel}];
    if (bytes <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

vd::GridView grid_view(const vd_grid *g, int elec_map, int desolv_map)
{
    vd::GridView v;
    v.ed = ed_for(g, elec_map, desolv_map);
    v.yz = v.ed ? g->d_yz : nullptr;
    v.maps = g->d_maps;
    v.n_maps = g->n_maps;
    v.nx = g->nx;
    v.ny = g->ny;
    v.nz = g->nz;
    v.mstride = (int64_t)g->nx * g->ny * g->nz;
    v.lo0 = g->lo[0]; v.lo1 = g->lo[1]; v.lo2 = g->lo[2];
    v.hi0 = g->hi[0]; v.hi1 = g->hi[1]; v.hi2 = g->hi[2];
    v.spacing = g->spacing;
    v.one = 1.0f;
    v.zpair = g->zpair ? 1 : 0;
    v.nyp = (g->ny + 1) / 2;
    v.tstride = g->tstride;
    return v;
}

/* Host-buffer pipeline: copy-in, kernel and copy-out each on their own stream, chained by
 * events over a ring of kRing staging slots, so the H2D engine (the e2e bound: 120 B of f64
 * genes per pose at ~54 GB/s) never waits for a kernel or a copy-out. */
constexpr int kRing = 3;
struct Pipe {
    cudaStream_t h, k, d;
    cudaEvent_t start, eh[kRing], ek[kRing], ed[kRing];
    /* staging slots, kept between calls (grown on demand) */
    char *in[kRing] = {};
    double *e[kRing] = {}, *a[kRing] = {};
    float *t[kRing] = {};
    size_t in_cap = 0;
    int64_t out_cap = 0;
};

/* Process-wide pool of pipes per device.  A call leases one for its duration, so
 * concurrent callers never share staging slots, and threads that come and go (the
 * reference's per-call worker pools) reuse pipes instead of leaking one each: the pool
 * holds at most as many pipes as calls ever ran at once on that device.  A pipe handed
 * back with copies still in flight is safe to reuse: its streams are in order and every
 * slot reuse waits on the slot's last events. */
class PipeLease {
  public:
    PipeLease()
    {
        cudaGetDevice(&dev_);
        {
            std::lock_guard<std::mutex> lk(mu());
            auto &fl = free_list()[dev_];
            if (!fl.empty()) {
                p_ = fl.back();
                fl.pop_back();
                return;
            }
        }
        p_ = new Pipe();
        cudaStreamCreateWithFlags(&p_->h, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&p_->k, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&p_->d, cudaStreamNonBlocking);
        for (int r = 0; r < kRing; ++r) {
            cudaEventCreateWithFlags(&p_->eh[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&p_->ek[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&p_->ed[r], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&p_->start, cudaEventDisableTiming);
        std::lock_guard<std::mutex> lk(mu());
        ++created()[dev_];
    }
    ~PipeLease()
    {
        std::lock_guard<std::mutex> lk(mu());
        free_list()[dev_].push_back(p_);
    }
    PipeLease(const PipeLease &) = delete;
    PipeLease &operator=(const PipeLease &) = delete;
    Pipe *operator->() const { return p_; }
    static int pipes_created(int dev)
    {
        std::lock_guard<std::mutex> lk(mu());
        return created()[dev];
    }

  private:
    static std::mutex &mu()
    {
        static std::mutex m;
        return m;
    }
    static std::map<int, std::vector<Pipe *>> &free_list()
    {
        static auto *m = new std::map<int, std::vector<Pipe *>>();  /* never destroyed: no CUDA calls at exit */
        return *m;
    }
    static std::map<int, int> &created()
    {
        static auto *m = new std::map<int, int>();
        return *m;
    }
    int dev_ = 0;
    Pipe *p_ = nullptr;
};
}  // namespace vdi

vd::LigView vd_ligands::view(int l) const
{
    vd::LigView v;
    const int a0 = atom_start[l], p0 = pair_start[l], t0 = tors_start[l];
    v.n_atoms = atom_start[l + 1] - a0;
    v.n_pairs = pair_start[l + 1] - p0;
    v.n_torsions = tors_start[l + 1] - t0;
    v.n_frag = n_frag[l];
    v.atom = d_atom + a0;
    v.atom2 = d_atom2 + a0;
    v.pij = d_pij + p0;
    v.pcoef = d_pcoef + p0;
    v.fcoef = d_fcoef + p0;
    v.fij = d_fij + p0;
    v.n_nohb = n_nohb[l];
    v.tors = d_tors + t0;
    v.frag = d_frag;
    v.tors32 = tors32[l];
    v.cut2 = cut2[l];
    v.penalty = penalty[l];
    v.elec_map = elec_map;
    v.desolv_map = desolv_map;
    return v;
}

using vdi::set_error;

extern "C" {

int vd_abi_version(void) { return VD_ABI_VERSION; }
const char *vd_last_error(void) { return vdi::g_err.c_str(); }

int vd_last_launch_count(int64_t *launches)
{
    *launches = vdi::g_launches;
    return 0;
}

int vd_pipe_count(int device)
{
    return vdi::PipeLease::pipes_created(device);
}

int vd_debug_check_flags(uint32_t *flags, int clear)
{
#ifdef VD_CHECKED
    if (clear < 0) {  /* self-test: each translation unit raises one known flag */
        vdi::chk_selftest_score();
        vdi::chk_selftest_ga();
    }
    VD_CK(cudaDeviceSynchronize());
    *flags = vdi::chk_flags_score(clear != 0) | vdi::chk_flags_ga(clear != 0);
    return 1;
#else
    (void)clear;
    *flags = 0;
    return 0;
#endif
}

int vd_device_count(int *count)
{
    *count = 0;
    VD_CK(cudaGetDeviceCount(count));
    return 0;
}

int vd_init(int device)
{
    VD_CK(cudaSetDevice(device));
    VD_CK(cudaFree(0));
    /* keep stream-ordered staging buffers in the pool between calls instead of
       returning them to the OS at every synchronisation */
    cudaMemPool_t pool;
    VD_CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    VD_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    return 0;
}

int vd_grid_create(const float *maps, int n_maps, int nx, int ny, int nz, const float lo[3],
                   const float hi[3], float spacing, vd_grid **out)
{
    *out = nullptr;
    if (n_maps < 1 || nx < 2 || ny < 2 || nz < 2 || !(spacing > 0.f)) {
        set_error("vd_grid_create: bad grid shape");
        return -1;
    }
    const size_t n = (size_t)n_maps * nx * ny * nz;
    if (n >= ((size_t)1 << 31)) {
        set_error("vd_grid_create: map stack exceeds 2^31 values");
        return -1;
    }
    vd_grid *g = new vd_grid();
    cudaGetDevice(&g->device);
    g->n_maps = n_maps;
    g->nx = nx; g->ny = ny; g->nz = nz;
    for (int k = 0; k < 3; ++k) { g->lo[k] = lo[k]; g->hi[k] = hi[k]; }
    g->spacing = spacing;
    if (!vdi::check(cudaMalloc(&g->d_maps, n * sizeof(float)), "cudaMalloc(maps)")) {
        delete g;
        return -1;
    }
    if (maps &&
        (!vdi::check(cudaMemcpy(g->d_maps, maps, n * sizeof(float), cudaMemcpyDefault), "upload maps") ||
         !vdi::make_packed(g))) {
        vd_grid_destroy(g);
        return -1;
    }
    *out = g;
    return 0;
}

int vd_grid_n_maps(const vd_grid *g) { return g ? g->n_maps : -1; }

int vd_grid_layout(const vd_grid *g)
{
    if (!g) return -1;
    return g->d_yz ? (g->zpair ? VD_LAYOUT_ZPAIR : VD_LAYOUT_BRICK) : VD_LAYOUT_PLAIN;
}

int vd_grid_download(const vd_grid *g, float *out)
{
    const size_t n = (size_t)g->n_maps * g->nx * g->ny * g->nz;
    VD_CK(cudaMemcpy(out, g->d_maps, n * sizeof(float), cudaMemcpyDefault));
    return 0;
}

int vd_grid_destroy(vd_grid *g)
{
    if (!g) return 0;
    cudaFree(g->d_maps);
    cudaFree(g->d_yz);
    for (auto &kv : g->d_ed) cudaFree(kv.second);
    delete g;
    return 0;
}

int vd_ligands_create(const vd_ligand_arrays *a, vd_ligands **out)
{
    *out = nullptr;
    const int L = a->n_ligands;
    if (L < 1) {
        set_error("vd_ligands_create: need at least one ligand");
        return -1;
    }
    const int NA = a->atom_start[L], NP = a->pair_start[L], NT = a->tors_start[L];
    int NF = 0;
    for (int t = 0; t < NT; ++t) NF = std::max(NF, a->frag_hi[t]);
    std::vector<float4> atom(std::max(NA, 1));
    std::vector<float2> atom2(std::max(NA, 1));
    std::vector<uint32_t> pij(std::max(NP, 1));
    std::vector<float4> pcoef(std::max(NP, 1));
    std::vector<int4> tors(std::max(NT, 1));
    std::vector<int> frag(std::max(NF, 1));
    auto *s = new vd_ligands();
    cudaGetDevice(&s->device);
    s->n_ligands = L;
    s->atom_start.assign(a->atom_start, a->atom_start + L + 1);
    s->pair_start.assign(a->pair_start, a->pair_start + L + 1);
    s->tors_start.assign(a->tors_start, a->tors_start + L + 1);
    s->elec_map = a->elec_map;
    s->desolv_map = a->desolv_map;
    s->max_atoms = s->max_torsions = 0;
    for (int l = 0; l < L; ++l) {
        const int a0 = a->atom_start[l], n = a->atom_start[l + 1] - a0;
        const int t0 = a->tors_start[l], T = a->tors_start[l + 1] - t0;
        if (n < 1 || n > 32767) {
            set_error("vd_ligands_create: ligand " + std::to_string(l) + " has " +
                      std::to_string(n) + " atoms (need 1..32767)");
            delete s;
            return -1;
        }
        s->max_atoms = std::max(s->max_atoms, n);
        s->max_torsions = std::max(s->max_torsions, T);
        s->n_frag.push_back(T ? a->frag_hi[t0 + T - 1] - a->frag_lo[t0] : 0);
        s->tors32.push_back(a->torsional32 ? a->torsional32[l] : 0.f);
        s->cut2.push_back(a->intra_cutoff2 ? a->intra_cutoff2[l] : INFINITY);
        s->penalty.push_back(a->penalty_scale ? a->penalty_scale[l] : 1.0e4f);
        for (int i = 0; i < n; ++i) {
            const int g = a0 + i;
            atom[g] = make_float4(a->centered0[3 * g], a->centered0[3 * g + 1],
                                  a->centered0[3 * g + 2], a->charge[g]);
            int m = a->atom_map[g];
            float mf;
            std::memcpy(&mf, &m, sizeof mf);
            atom2[g] = make_float2(a->desolv_factor[g], mf);
        }
        for (int k = a->pair_start[l]; k < a->pair_start[l + 1]; ++k) {
            const int i = a->pair_i[k], j = a->pair_j[k];
            if (i < 0 || j < 0 || i >= n || j >= n) {
                set_error("vd_ligands_create: pair atom index out of range");
                delete s;
                return -1;
            }
            pij[k] = (uint32_t)i | ((uint32_t)j << 15) | ((a->pair_hb[k] ? 1u : 0u) << 31);
            pcoef[k] = make_float4(a->pair_a[k], a->pair_b[k], a->pair_qq[k], a->pair_desolv[k]);
        }
        for (int t = t0; t < t0 + T; ++t) {
            if (a->axis_a[t] < 0 || a->axis_a[t] >= n || a->axis_b[t] < 0 || a->axis_b[t] >= n ||
                a->frag_lo[t] < 0 || a->frag_hi[t] < a->frag_lo[t]) {
                set_error("vd_ligands_create: bad torsion record");
                delete s;
                return -1;
            }
            tors[t] = make_int4(a->axis_a[t], a->axis_b[t], a->frag_lo[t], a->frag_hi[t]);
            for (int f = a->frag_lo[t]; f < a->frag_hi[t]; ++f) {
                if (a->frag_index[f] < 0 || a->frag_index[f] >= n) {
                    set_error("vd_ligands_create: fragment atom index out of range");
                    delete s;
                    return -1;
                }
                frag[f] = a->frag_index[f];
            }
        }
    }
    /* fast order: stable partition by the 12-10 flag (one hb-uniform stream each) */
    std::vector<float4> fcoef(std::max(NP, 1));
    std::vector<int2> fij(std::max(NP, 1));  /* 3*i, 3*j (PairTile::off) */
    for (int l = 0; l < L; ++l) {
        const int p0 = a->pair_start[l], p1 = a->pair_start[l + 1];
        int w = p0;
        for (int g = 0; g < 2; ++g) {
            if (g == 1) s->n_nohb.push_back(w - p0);
            for (int k = p0; k < p1; ++k)
                if ((a->pair_hb[k] ? 1 : 0) == g) {
                    fcoef[w] = pcoef[k];
                    fij[w] = make_int2(3 * a->pair_i[k], 3 * a->pair_j[k]);
                    ++w;
                }
        }
    }
    bool ok = vdi::check(cudaMalloc(&s->d_atom, atom.size() * sizeof(float4)), "alloc atoms") &&
              vdi::check(cudaMalloc(&s->d_atom2, atom2.size() * sizeof(float2)), "alloc atoms2") &&
              vdi::check(cudaMalloc(&s->d_pij, pij.size() * sizeof(uint32_t)), "alloc pairs") &&
              vdi::check(cudaMalloc(&s->d_pcoef, pcoef.size() * sizeof(float4)), "alloc coef") &&
              vdi::check(cudaMalloc(&s->d_tors, tors.size() * sizeof(int4)), "alloc tors") &&
              vdi::check(cudaMalloc(&s->d_frag, frag.size() * sizeof(int)), "alloc frag") &&
              vdi::check(cudaMemcpy(s->d_atom, atom.data(), atom.size() * sizeof(float4), cudaMemcpyHostToDevice), "up atoms") &&
              vdi::check(cudaMemcpy(s->d_atom2, atom2.data(), atom2.size() * sizeof(float2), cudaMemcpyHostToDevice), "up atoms2") &&
              vdi::check(cudaMemcpy(s->d_pij, pij.data(), pij.size() * sizeof(uint32_t), cudaMemcpyHostToDevice), "up pairs") &&
              vdi::check(cudaMemcpy(s->d_pcoef, pcoef.data(), pcoef.size() * sizeof(float4), cudaMemcpyHostToDevice), "up coef") &&
              vdi::check(cudaMemcpy(s->d_tors, tors.data(), tors.size() * sizeof(int4), cudaMemcpyHostToDevice), "up tors") &&
              vdi::check(cudaMemcpy(s->d_frag, frag.data(), frag.size() * sizeof(int), cudaMemcpyHostToDevice), "up frag") &&
              vdi::check(cudaMalloc(&s->d_fcoef, fcoef.size() * sizeof(float4)), "alloc fcoef") &&
              vdi::check(cudaMalloc(&s->d_fij, fij.size() * sizeof(int2)), "alloc fij") &&
              vdi::check(cudaMemcpy(s->d_fcoef, fcoef.data(), fcoef.size() * sizeof(float4), cudaMemcpyHostToDevice), "up fcoef") &&
              vdi::check(cudaMemcpy(s->d_fij, fij.data(), fij.size() * sizeof(int2), cudaMemcpyHostToDevice), "up fij");
    if (!ok) {
        vd_ligands_destroy(s);
        return -1;
    }
    *out = s;
    return 0;
}

int vd_ligands_n_torsions(const vd_ligands *s, int lig)
{
    if (!s || lig < 0 || lig >= s->n_ligands) return -1;
    return s->tors_start[lig + 1] - s->tors_start[lig];
}

int vd_ligands_destroy(vd_ligands *s)
{
    if (!s) return 0;
    cudaFree(s->d_atom);
    cudaFree(s->d_atom2);
    cudaFree(s->d_pij);
    cudaFree(s->d_pcoef);
    cudaFree(s->d_tors);
    cudaFree(s->d_frag);
    cudaFree(s->d_fcoef);
    cudaFree(s->d_fij);
    delete s;
    return 0;
}

/* Shared driver of vd_score_genes / vd_score_poses. */
static int score_common(const vd_grid *g, const vd_ligands *s, int lig, const void *in,
                        bool in_is_genes, int64_t P, double *inter, double *intra, float *total,
                        int mode, void *stream)
{
    if (!g || !s || lig < 0 || lig >= s->n_ligands) {
        set_error("vd_score: bad grid/ligand handle or index");
        return -1;
    }
    if (P <= 0) return 0;
    if (!in || !inter || !intra) {
        set_error("vd_score: null input/output");
        return -1;
    }
    const vd::LigView L = s->view(lig);
    const vd::GridView G = vdi::grid_view(g, s->elec_map, s->desolv_map);
    const int ngenes = 7 + L.n_torsions;
    const size_t in_row = in_is_genes ? sizeof(double) * ngenes : sizeof(float) * 3 * L.n_atoms;
    const int src = in_is_genes ? 0 : 1;
    cudaStream_t cs = (cudaStream_t)stream;
    const bool in_dev = vdi::is_device_ptr(in);
    const bool oe = vdi::is_device_ptr(inter), oa = vdi::is_device_ptr(intra),
               ot = total ? vdi::is_device_ptr(total) : true;
    if (in_dev && oe && oa && ot) {
        VD_CK(vd::launch_score(mode, src, G, L, in_is_genes ? (const double *)in : nullptr,
                               in_is_genes ? nullptr : (const float *)in, P, ngenes, inter, intra,
                               total, cs));
        return 0;
    }
    /* chunked pipeline through a ring of device staging slots (see Pipe).  Chunks of CH
       poses, the last CH split in halves and quarters so the final kernel + copy-out that
       trail the last copy-in are short. */
    vdi::PipeLease pp;
    static const int64_t chunk_env = getenv("VD_CHUNK") ? atoll(getenv("VD_CHUNK")) : 0;
    const int64_t CH = std::min<int64_t>(P, chunk_env > 0 ? chunk_env : (1 << 17));
    std::vector<std::pair<int64_t, int64_t>> chunks;  /* (offset, count) */
    {
        int64_t off = 0;
        while (P - off > CH) {
            chunks.push_back({off, CH});
            off += CH;
        }
        int64_t rest = P - off, piece = std::max<int64_t>(CH / 2, 1);
        while (rest > 0) {
            const int64_t n = rest > piece && piece >= 4096 ? piece : rest;
            chunks.push_back({off, n});
            off += n;
            rest -= n;
            piece /= 2;
        }
    }
    VD_CK(cudaEventRecord(pp->start, cs));
    VD_CK(cudaStreamWaitEvent(pp->h, pp->start, 0));
    VD_CK(cudaStreamWaitEvent(pp->k, pp->start, 0));
    VD_CK(cudaStreamWaitEvent(pp->d, pp->start, 0));
    if ((!in_dev && (size_t)CH * in_row > pp->in_cap) || ((!oe || !oa || !ot) && CH > pp->out_cap)) {
        /* grow the slots: drain whatever still uses the old ones */
        VD_CK(cudaStreamSynchronize(pp->h));
        VD_CK(cudaStreamSynchronize(pp->k));
        VD_CK(cudaStreamSynchronize(pp->d));
        if (!in_dev && (size_t)CH * in_row > pp->in_cap) {
            for (int r = 0; r < vdi::kRing; ++r) {
                cudaFree(pp->in[r]);
                pp->in[r] = nullptr;
            }
            pp->in_cap = 0;
            for (int r = 0; r < vdi::kRing; ++r) VD_CK(cudaMalloc((void **)&pp->in[r], CH * in_row));
            pp->in_cap = (size_t)CH * in_row;
        }
        if ((!oe || !oa || !ot) && CH > pp->out_cap) {
            for (int r = 0; r < vdi::kRing; ++r) {
                cudaFree(pp->e[r]); cudaFree(pp->a[r]); cudaFree(pp->t[r]);
                pp->e[r] = pp->a[r] = nullptr;
                pp->t[r] = nullptr;
            }
            pp->out_cap = 0;
            for (int r = 0; r < vdi::kRing; ++r) {
                VD_CK(cudaMalloc((void **)&pp->e[r], CH * sizeof(double)));
                VD_CK(cudaMalloc((void **)&pp->a[r], CH * sizeof(double)));
                VD_CK(cudaMalloc((void **)&pp->t[r], CH * sizeof(float)));
            }
            pp->out_cap = CH;
        }
    }
    char **d_in = pp->in;
    double **d_e = pp->e, **d_a = pp->a;
    float **d_t = pp->t;
    int rc = 0;
    for (size_t c = 0; c < chunks.size() && rc == 0; ++c) {
        const int r = (int)(c % vdi::kRing);
        const int64_t off = chunks[c].first, n = chunks[c].second;
        const char *src_in = (const char *)in + off * in_row;
        const void *kin = src_in;
        if (!in_dev) {
            /* slot r's previous kernel (chunk c - kRing) has read its input */
            if (!vdi::check(cudaStreamWaitEvent(pp->h, pp->ek[r], 0), "wait k") ||
                !vdi::check(cudaMemcpyAsync(d_in[r], src_in, n * in_row, cudaMemcpyHostToDevice, pp->h), "H2D") ||
                !vdi::check(cudaEventRecord(pp->eh[r], pp->h), "event h") ||
                !vdi::check(cudaStreamWaitEvent(pp->k, pp->eh[r], 0), "wait h")) { rc = -1; break; }
            kin = d_in[r];
        }
        double *ke = oe ? inter + off : d_e[r];
        double *ka = oa ? intra + off : d_a[r];
        float *kt = total ? (ot ? total + off : d_t[r]) : nullptr;
        /* slot r's previous copy-out (chunk c - kRing) has drained its outputs */
        if (!vdi::check(cudaStreamWaitEvent(pp->k, pp->ed[r], 0), "wait d") ||
            !vdi::check(vd::launch_score(mode, src, G, L, in_is_genes ? (const double *)kin : nullptr,
                                         in_is_genes ? nullptr : (const float *)kin, n, ngenes, ke, ka, kt, pp->k),
                        "score kernel") ||
            !vdi::check(cudaEventRecord(pp->ek[r], pp->k), "event k") ||
            !vdi::check(cudaStreamWaitEvent(pp->d, pp->ek[r], 0), "wait k")) { rc = -1; break; }
        if ((!oe && !vdi::check(cudaMemcpyAsync(inter + off, ke, n * sizeof(double), cudaMemcpyDeviceToHost, pp->d), "D2H e")) ||
            (!oa && !vdi::check(cudaMemcpyAsync(intra + off, ka, n * sizeof(double), cudaMemcpyDeviceToHost, pp->d), "D2H a")) ||
            (total && !ot && !vdi::check(cudaMemcpyAsync(total + off, kt, n * sizeof(float), cudaMemcpyDeviceToHost, pp->d), "D2H t")) ||
            !vdi::check(cudaEventRecord(pp->ed[r], pp->d), "event d")) { rc = -1; break; }
    }
    /* join: the caller's stream waits for all three pipeline streams */
    cudaEventRecord(pp->eh[0], pp->h);
    cudaStreamWaitEvent(pp->d, pp->eh[0], 0);
    cudaEventRecord(pp->ek[0], pp->k);
    cudaStreamWaitEvent(pp->d, pp->ek[0], 0);
    cudaEventRecord(pp->ed[0], pp->d);
    cudaStreamWaitEvent(cs, pp->ed[0], 0);
    if (rc) return rc;
    if (!(oe && oa && ot)) VD_CK(cudaStreamSynchronize(pp->d));
    return 0;
}

int vd_score_genes(const vd_grid *g, const vd_ligands *s, int lig, const double *genes,
                   int64_t P, double *inter, double *intra, float *total, int mode, void *stream)
{
    return score_common(g, s, lig, genes, true, P, inter, intra, total, mode, stream);
}

int vd_score_poses(const vd_grid *g, const vd_ligands *s, int lig, const float *poses,
                   int64_t P, double *inter, double *intra, int mode, void *stream)
{
    return score_common(g, s, lig, poses, false, P, inter, intra, nullptr, mode, stream);
}

static int pose_common(const vd_ligands *s, int lig, const double *genes, int64_t P, float *poses,
                       void *stream, int tpp)
{
    if (!s || lig < 0 || lig >= s->n_ligands) {
        set_error("vd_pose_genes: bad ligand handle or index");
        return -1;
    }
    if (P <= 0) return 0;
    const vd::LigView L = s->view(lig);
    const int ngenes = 7 + L.n_torsions;
    cudaStream_t st = (cudaStream_t)stream;
    const double *dg = genes;
    float *dp = poses;
    const bool gin = vdi::is_device_ptr(genes), pout = vdi::is_device_ptr(poses);
    if (!gin) {
        VD_CK(cudaMallocAsync((void **)&dg, P * ngenes * sizeof(double), st));
        VD_CK(cudaMemcpyAsync((void *)dg, genes, P * ngenes * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    if (!pout) VD_CK(cudaMallocAsync((void **)&dp, P * 3 * L.n_atoms * sizeof(float), st));
    VD_CK(vd::launch_pose(L, dg, P, ngenes, dp, st, tpp));
    if (!pout) {
        VD_CK(cudaMemcpyAsync(poses, dp, P * 3 * L.n_atoms * sizeof(float), cudaMemcpyDeviceToHost, st));
        VD_CK(cudaFreeAsync(dp, st));
    }
    if (!gin) VD_CK(cudaFreeAsync((void *)dg, st));
    if (!pout) VD_CK(cudaStreamSynchronize(st));
    return 0;
}

int vd_pose_genes(const vd_ligands *s, int lig, const double *genes, int64_t P, float *poses,
                  void *stream)
{
    return pose_common(s, lig, genes, P, poses, stream, 0);
}

int vd_debug_pose_genes(const vd_ligands *s, int lig, const double *genes, int64_t P, int tpp,
                        float *poses)
{
    if (tpp != 4 && tpp != 8 && tpp != 16) {
        set_error("vd_debug_pose_genes: tpp must be 4, 8 or 16");
        return -1;
    }
    return pose_common(s, lig, genes, P, poses, nullptr, tpp);
}

}  // extern "C"
