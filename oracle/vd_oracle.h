/* vd_oracle.h -- private header of the CPU oracle (test infrastructure only;
 * see vd_oracle.c). */
#ifndef VD_ORACLE_H
#define VD_ORACLE_H
#include <stdint.h>

typedef struct {
    /* grid: maps[(m*nx + ix)*ny + iy)*nz + iz], C order, z fastest */
    const float *maps;
    int nx, ny, nz;
    float lo[3], hi[3], spacing, penalty;
    /* per atom */
    int n_atoms;
    const int32_t *atom_map;   /* map index of the atom's type map */
    int elec_map, desolv_map;
    const float *charge, *dsf;
    /* pairs */
    int n_pairs;
    const int32_t *pi, *pj;
    const float *pa, *pb, *pqq, *pdsl;
    const uint8_t *phb;
    float cut2;
    int lane;                  /* simd lane width (DEFAULT_LANE = 8) */
    /* pose */
    const float *centered0;    /* (3, n) */
    int n_torsions;
    const int32_t *frag_start, *frag_index, *axis_a, *axis_b;
} or_ligand;

void or_pose_into(const or_ligand *L, const double *g, float *px, float *py, float *pz);
double or_inter_one(const or_ligand *L, const float *px, const float *py, const float *pz);
double or_intra_one(const or_ligand *L, const float *px, const float *py, const float *pz);
float or_total32(double inter, double intra, float tors);

#endif
