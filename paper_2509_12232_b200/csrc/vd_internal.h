/* vd_internal.h -- handle layouts and helpers shared by the .cu files of libvdb200. */
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "vd_device.cuh"
#include "vecdock_b200.h"

struct vd_grid {
    int device;
    int n_maps, nx, ny, nz;
    float lo[3], hi[3], spacing;
    float *d_maps;           /* (n_maps, nx, ny, nz) */
    float4 *d_yz;            /* packed type maps (yz-bricks or z-pairs), or null (see GridView) */
    bool zpair;              /* d_yz holds zy z-pairs (8 B/node) instead of yz-bricks (16 B/node) */
    int64_t tstride;         /* elements per packed type map */
    std::vector<char> yz_packed;
    std::mutex ed_lock;
    std::map<std::pair<int, int>, float4 *> d_ed;  /* packed (elec, desolv) per map pair */
};

struct vd_ligands {
    int device;
    int n_ligands;
    std::vector<int> atom_start, pair_start, tors_start;  /* host copies of the CSR */
    std::vector<float> tors32, cut2, penalty;
    int elec_map, desolv_map;
    int max_atoms, max_torsions;
    float4 *d_atom;
    float2 *d_atom2;
    uint32_t *d_pij;
    float4 *d_pcoef;
    int4 *d_tors;
    int *d_frag;
    float4 *d_fcoef;          /* fast-order pairs: 12-6 then 12-10 */
    int2 *d_fij;              /* 3*i, 3*j */
    std::vector<int> n_nohb, n_frag;
    vd::LigView view(int lig) const;
};

namespace vdi {
void set_error(const std::string &msg);
bool check(cudaError_t e, const char *what);
void set_detail(const std::string &msg);  /* reason attached to the next failed check() */
bool is_device_ptr(const void *p);
extern thread_local int64_t g_launches;
vd::GridView grid_view(const vd_grid *g, int elec_map, int desolv_map);
/* Raise a kernel's dynamic shared-memory limit to at least `bytes` on the current device.
 * The attribute is process-wide, so it only ever grows: a thread launching a smaller ligand
 * must not lower the limit another thread's launch of the same kernel relies on. */
cudaError_t raise_smem_limit(const void *kernel, unsigned bytes);
bool make_packed(vd_grid *g);
/* checked build: the device check-flag word of each translation unit (0 otherwise) */
unsigned chk_flags_score(bool clear);
unsigned chk_flags_ga(bool clear);
void chk_selftest_score();  /* raise one flag per translation unit (checked build) */
void chk_selftest_ga();

}  // namespace vdi

namespace vd {
/* wide: the score kernels' rule (256-thread CTAs whatever the pose tile); the persistent GA
 * kernels keep 4 subs up to 96 atoms */
int pick_shape(int n_atoms, int n_pairs, int n_tors, bool exact, int *npp, int *tpp, bool wide = false);
}

#define VD_CK(call)                                        \
    do {                                                   \
        if (!vdi::check((call), #call)) return -1;         \
    } while (0)
