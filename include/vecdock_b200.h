/*
 * vecdock_b200.h -- C-ABI of the B200 docking hot path (libvdb200.so).
 *
 * Plain C types only.  Every entry returns 0 on success and < 0 on error,
 * with a thread-local message in vd_last_error().  Pointers passed for bulk
 * inputs/outputs may be host memory (pageable or pinned) or device memory
 * (e.g. torch tensors' data_ptr()); the library detects which.  A call with
 * any host output synchronises its stream before returning; an all-device
 * call is asynchronous on `stream` (NULL = legacy default stream).
 *
 * Each entry replaces one reference seam (paths under
 * /root/reference/pkg/src/vecdock):
 *
 *   vd_grid_load_mugd                 grids.py:269-303 read_grid_set (MUGD file -> device)
 *   vd_grid_create / vd_grid_build    grids.py:83-119 GridMapSet, grids.py:122-202
 *                                     build_grid_maps; the map stack of
 *                                     scoring/__init__.py:158-161 becomes one
 *                                     shared device copy indexed per atom
 *   vd_ligands_create                 scoring/__init__.py:133-207 prepare_context
 *                                     (ScoringContext fields, CSR over ligands)
 *   vd_score_genes                    SimdBackend.dock_population
 *                                     (scoring/simd.py:294-311) + the total32
 *                                     rounding of scoring/__init__.py:345
 *   vd_score_poses                    SimdBackend.score_many (scoring/simd.py:277-292),
 *                                     inter_one/intra_one with P = 1 (:250-275)
 *   vd_pose_genes                     pose.pose_population (pose.py:137-205)
 *   vd_dock_batch                     ga.dock (ga.py:180-235) for every ligand of a
 *                                     screen_batch (screening.py:165-244), GA on device
 */
#ifndef VECDOCK_B200_H
#define VECDOCK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VD_ABI_VERSION 1

typedef struct vd_grid vd_grid;
typedef struct vd_ligands vd_ligands;

/* numerics of the energy stage (the pose stage is always bit-exact) */
enum vd_mode {
    VD_MODE_FAST = 0,  /* fp32 MUFU/FMA pair & lerp math, fp32 partials -> fp64 sums */
    VD_MODE_EXACT = 1  /* the reference's canonical f32/f64 sequences and fp64
                          summation order (scoring/reference.py:11-35, simd lane 8) */
};

int vd_abi_version(void);
const char *vd_last_error(void);
int vd_device_count(int *count);
int vd_init(int device); /* select `device` for the calling thread, create its context */

/* ---- grid maps (shared, read-only constant data) ------------------------ */
/* maps: (n_maps, nx, ny, nz) f32, C order (z fastest), host or device. */
int vd_grid_create(const float *maps, int n_maps, int nx, int ny, int nz, const float lo[3],
                   const float hi[3], float spacing, vd_grid **out);

typedef struct {
    double r_eq, eps, volume, solpar;
    int32_t donor, acceptor;
} vd_atom_type;

typedef struct {
    double vdw, hbond, elec, desolv;
} vd_weights;

/* AutoGrid-style build on the device: probe maps (in `probe` order), then
 * @elec, then @desolv; fp64 per-node sums over receptor atoms in order. */
int vd_grid_build(const float *rec_xyz /* (3, n_rec) */, const int32_t *rec_type,
                  const float *rec_charge, int n_rec, const vd_atom_type *table, int n_types,
                  const int32_t *probe, int n_probe, const double origin[3], double spacing,
                  int nx, int ny, int nz, const vd_weights *w, double cutoff, vd_grid **out);
int vd_grid_n_maps(const vd_grid *g);
/* gather layout chosen at creation: plain maps only, type maps as
 * yz-bricks, or as z-pairs (both with elec/desolv bricks); -1 for a NULL handle */
enum vd_layout { VD_LAYOUT_PLAIN = 0, VD_LAYOUT_BRICK = 1, VD_LAYOUT_ZPAIR = 2 };
int vd_grid_layout(const vd_grid *g);
int vd_grid_download(const vd_grid *g, float *out /* (n_maps, nx, ny, nz) host */);

/* MUGD grid files (vd/grids.py:232-303 write_grid_set / read_grid_set): payloads are
 * read into pinned host staging, copied as stored (x fastest) and transposed on the
 * device into the z-fastest stack; maps keep file order.  Format errors return -2 with
 * the reference's GridFormatError message in vd_last_error(); other failures -1.
 * vd_mugd_read_header fills `info` and, when `labels` is non-null, the map labels as
 * consecutive NUL-terminated strings (info->labels_bytes in total). */
typedef struct {
    int32_t n_maps, nx, ny, nz;
    float origin[3];
    float spacing;
    int32_t labels_bytes;
} vd_mugd_info;
int vd_mugd_read_header(const char *path, vd_mugd_info *info, char *labels, int labels_cap);
int vd_grid_load_mugd(const char *path, vd_grid **out);
int vd_grid_destroy(vd_grid *g);

/* ---- ligand set (ScoringContext records, CSR over L ligands) ------------- */
typedef struct {
    int32_t n_ligands;
    const int32_t *atom_start;   /* [L+1] */
    const int32_t *pair_start;   /* [L+1] */
    const int32_t *tors_start;   /* [L+1] */
    const float *centered0;      /* [sumN][3] pose_centered0, atom-major */
    const float *charge;         /* [sumN] */
    const float *desolv_factor;  /* [sumN] */
    const int32_t *atom_map;     /* [sumN] grid map index of each atom's type map */
    const int32_t *pair_i;       /* [sumP] ligand-local atom indices */
    const int32_t *pair_j;
    const float *pair_a, *pair_b, *pair_qq, *pair_desolv; /* [sumP] weight-folded */
    const uint8_t *pair_hb;      /* [sumP] 12-10 flag */
    const int32_t *axis_a;       /* [sumT] ligand-local */
    const int32_t *axis_b;
    const int32_t *frag_lo;      /* [sumT] absolute offsets into frag_index */
    const int32_t *frag_hi;
    const int32_t *frag_index;   /* [sumF] ligand-local atom indices */
    const float *torsional32;    /* [L] f32(w_tors * T) */
    const float *intra_cutoff2;  /* [L] (inf = none) */
    const float *penalty_scale;  /* [L] out-of-box penalty (1e4) */
    int32_t elec_map, desolv_map;
} vd_ligand_arrays;

int vd_ligands_create(const vd_ligand_arrays *a, vd_ligands **out);
int vd_ligands_n_torsions(const vd_ligands *s, int lig);
int vd_ligands_destroy(vd_ligands *s);

/* ---- scoring ------------------------------------------------------------ */
/* genes: (P, 7 + T) f64 row-major; inter/intra f64 [P]; total f32 [P] (nullable). */
int vd_score_genes(const vd_grid *g, const vd_ligands *s, int lig, const double *genes,
                   int64_t P, double *inter, double *intra, float *total, int mode,
                   void *stream);
/* poses: (P, 3, N) f32. */
int vd_score_poses(const vd_grid *g, const vd_ligands *s, int lig, const float *poses,
                   int64_t P, double *inter, double *intra, int mode, void *stream);
int vd_pose_genes(const vd_ligands *s, int lig, const double *genes, int64_t P,
                  float *poses /* (P, 3, N) */, void *stream);

/* ---- GA docking on device ------------------------------------------------ */
typedef struct {
    int32_t pop, generations, tournament, elitism;
    double cx_rate, mut_rate, sigma_t, sigma_r, sigma_tor;
    double lo[3], hi[3]; /* translation bounds (the grid box) */
} vd_ga_params;

/* Dock ligands [first, first + count) of the set; ligand l uses Philox key
 * (seed, lig_index_base + l).  Outputs are indexed by l - first. */
int vd_dock_batch(const vd_grid *g, const vd_ligands *s, int first, int count,
                  const vd_ga_params *p, uint64_t seed, int64_t lig_index_base, int mode,
                  float *best_total, double *best_inter, double *best_intra,
                  double *best_genes /* [count][gstride] */, int gstride,
                  float *trace /* nullable [count][generations + 1] */, int64_t *n_evals,
                  void *stream);

/* ---- batched host preprocessing (no device needed) ----------------------- */
/* Restates build_nonbond_pairlist / build_fragment_masks / prepare_context
 * (vd/model.py:174-269, vd/scoring/__init__.py:117-207) bit for bit for many
 * ligands (OpenMP).  Pass 1 sizes the CSR; pass 2 fills vd_ligand_arrays fields.
 * xyz is (3, n) per ligand at 3*atom_start[l]; bonds/axes are index pairs. */
int vd_prepare_count(int n_ligands, const int32_t *atom_start, const float *xyz,
                     const int32_t *bond_start, const int32_t *bonds, const int32_t *tors_start,
                     const int32_t *axes, int64_t *n_pairs, int64_t *n_frag);
int vd_prepare_fill(int n_ligands, const int32_t *atom_start, const float *xyz,
                    const int32_t *type_index, const float *charge, const int32_t *bond_start,
                    const int32_t *bonds, const int32_t *tors_start, const int32_t *axes,
                    const vd_atom_type *table, int n_types, const int32_t *type_map,
                    const vd_weights *w, double w_tors, const int64_t *pair_start,
                    const int64_t *frag_start, float *centered0, float *dsf, int32_t *atom_map,
                    int32_t *pair_i, int32_t *pair_j, float *pair_a, float *pair_b,
                    float *pair_qq, float *pair_dsl, uint8_t *pair_hb, int32_t *frag_lo,
                    int32_t *frag_hi, int32_t *frag_index, float *torsional32);

/* Synthetic cfg2/3/4 ligands, counter-keyed per index. */
int vd_synth_count(uint64_t seed, int64_t first, int count, int h_lo, int h_hi, double hd_ratio,
                   int t_lo, int t_hi, int32_t *n_atoms, int32_t *n_tors_max);
int vd_synth_fill(uint64_t seed, int64_t first, int count, int h_lo, int h_hi, double hd_ratio,
                  int t_lo, int t_hi, const int32_t *heavy_types, int32_t hd_type,
                  const int32_t *atom_start, float *xyz, int32_t *type_index, float *charge,
                  int32_t *bonds, int32_t *n_tors, int32_t *axes);

/* device-side counters of the last call on this thread (kernel launches) */
int vd_last_launch_count(int64_t *launches);
/* staging pipelines (3 streams + ring slots) ever created on `device`: host-buffer calls
 * lease one from a process-wide pool, so this is the peak number of concurrent calls,
 * not the number of threads that ever called */
int vd_pipe_count(int device);
/* checked build (libvdb200_checked.so, -DVD_CHECKED): OR of the device bounds/invariant
 * flags raised since the last clear (bit = site, csrc/vd_device.cuh VD_SITE_*); returns 1.
 * clear < 0 first runs a self-test that raises VD_SITE_TILE and VD_SITE_POP (bits 6, 5)
 * from the score and GA translation units, then reads and clears.
 * The production build returns 0 and *flags = 0. */
int vd_debug_check_flags(uint32_t *flags, int clear);

/* ---- test probes (parity checks of the GA's device randomness) ------------
 * They run the GA kernel's own device functions on chosen inputs, so the
 * oracle (oracle/or_rng.c, oracle/vd_ga_oracle.c) can check them draw for draw.
 * Counter map: block (slot/4, idx, gen, phase), word slot%4.
 * (vd_debug_pose_genes, below, does the same for the fast score kernel's pose stage.)
 *   vd_debug_rng kind 0: uint64 words [n_idx][n_slot] of (phase, gen);
 *                kind 1: f64 normals [n_idx][n_slot], component = slot
 *   vd_debug_ga_init:  init_population (vd/ga.py:90-109) -> [pop][7+T]
 *   vd_debug_ga_breed: the pop - elitism bred children of next_generation
 *                      (vd/ga.py:139-174) -> [pop - elitism][7+T]
 * All buffers are host memory; the calls synchronise. */
int vd_debug_rng(int kind, uint64_t seed, uint64_t lig_index, int phase, int64_t gen,
                 int64_t n_idx, int n_slot, void *out);
int vd_debug_ga_init(const vd_ga_params *p, int n_torsions, uint64_t seed, uint64_t lig_index,
                     double *out);
int vd_debug_ga_breed(const vd_ga_params *p, int n_torsions, const double *cur,
                      const float *fitness, int gen, uint64_t seed, uint64_t lig_index,
                      double *children);
/* the fast score kernel's pose stage (pose tile of TPP = 4, 8 or 16 sub-threads per pose pair,
 * shared scratch, barrier-ordered torsion chain) written out as (P, 3, N) f32 poses */
int vd_debug_pose_genes(const vd_ligands *s, int lig, const double *genes, int64_t P, int tpp,
                        float *poses);

#ifdef __cplusplus
}
#endif
#endif /* VECDOCK_B200_H */
