/*
 * vd_score.cu -- fused pose + inter + intra scoring kernels (thread per pose).
 *
 * One launch scores P genotypes (or given poses) of ONE ligand:
 * SimdBackend.dock_population / score_many semantics
 * (vd/scoring/simd.py:141-154, 225-240, 277-311) plus the total32 rounding of
 * vd/scoring/__init__.py:345.  See vd_device.cuh for the stage contracts.
 */
#include "vd_internal.h"

namespace vd {

enum { SRC_GENES = 0, SRC_POSES = 1 };

template <bool EXACT, int B, int SRC>
__global__ void __launch_bounds__(B) score_kernel(GridView G, LigView L,
                                                  const double *__restrict__ genes,
                                                  const float *__restrict__ poses, int64_t P,
                                                  int ngenes, double *__restrict__ inter,
                                                  double *__restrict__ intra,
                                                  float *__restrict__ total)
{
    extern __shared__ float smem[];
    const int64_t p = (int64_t)blockIdx.x * B + threadIdx.x;
    if (p >= P) return;
    float *S = smem + threadIdx.x;
    if (SRC == SRC_GENES) {
        build_pose<B>(L, genes + p * ngenes, S);
    } else {
        const float *src = poses + p * 3 * L.n_atoms;
        for (int i = 0; i < L.n_atoms; ++i) {
            VD_S(i, 0) = src[i];
            VD_S(i, 1) = src[L.n_atoms + i];
            VD_S(i, 2) = src[2 * L.n_atoms + i];
        }
    }
    const double e = inter_energy<EXACT, B>(L, G, S);
    const double a = L.n_pairs ? intra_energy<EXACT, B>(L, S) : 0.0;
    inter[p] = e;
    intra[p] = a;
    if (total) total[p] = total32(e, a, L.tors32);
}

template <int B>
__global__ void __launch_bounds__(B) pose_kernel(LigView L, const double *__restrict__ genes,
                                                 int64_t P, int ngenes, float *__restrict__ out)
{
    extern __shared__ float smem[];
    const int64_t p = (int64_t)blockIdx.x * B + threadIdx.x;
    if (p >= P) return;
    float *S = smem + threadIdx.x;
    build_pose<B>(L, genes + p * ngenes, S);
    float *dst = out + p * 3 * L.n_atoms;
    for (int i = 0; i < L.n_atoms; ++i) {
        dst[i] = VD_S(i, 0);
        dst[L.n_atoms + i] = VD_S(i, 1);
        dst[2 * L.n_atoms + i] = VD_S(i, 2);
    }
}

template <bool EXACT, int B, int SRC>
static cudaError_t launch_score_t(const GridView &G, const LigView &L, const double *genes,
                                  const float *poses, int64_t P, int ngenes, double *inter,
                                  double *intra, float *total, cudaStream_t st)
{
    const size_t smem = sizeof(float) * 3 * (size_t)L.n_atoms * B;
    auto k = score_kernel<EXACT, B, SRC>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (P + B - 1) / B;
    k<<<(unsigned)blocks, B, smem, st>>>(G, L, genes, poses, P, ngenes, inter, intra, total);
    ++vdi::g_launches;
    return cudaGetLastError();
}

template <bool EXACT, int SRC>
static cudaError_t launch_score_m(int B, const GridView &G, const LigView &L, const double *genes,
                                  const float *poses, int64_t P, int ngenes, double *inter,
                                  double *intra, float *total, cudaStream_t st)
{
    switch (B) {
    case 128: return launch_score_t<EXACT, 128, SRC>(G, L, genes, poses, P, ngenes, inter, intra, total, st);
    case 64: return launch_score_t<EXACT, 64, SRC>(G, L, genes, poses, P, ngenes, inter, intra, total, st);
    default: return launch_score_t<EXACT, 32, SRC>(G, L, genes, poses, P, ngenes, inter, intra, total, st);
    }
}

cudaError_t launch_score(int mode, int src, const GridView &G, const LigView &L,
                         const double *genes, const float *poses, int64_t P, int ngenes,
                         double *inter, double *intra, float *total, cudaStream_t st)
{
    int B;
    if (vdi::pick_block(L.n_atoms, &B)) return cudaErrorInvalidValue;
    if (P <= 0) return cudaSuccess;
    if (mode == VD_MODE_EXACT)
        return src == SRC_GENES
                   ? launch_score_m<true, SRC_GENES>(B, G, L, genes, poses, P, ngenes, inter, intra, total, st)
                   : launch_score_m<true, SRC_POSES>(B, G, L, genes, poses, P, ngenes, inter, intra, total, st);
    return src == SRC_GENES
               ? launch_score_m<false, SRC_GENES>(B, G, L, genes, poses, P, ngenes, inter, intra, total, st)
               : launch_score_m<false, SRC_POSES>(B, G, L, genes, poses, P, ngenes, inter, intra, total, st);
}

cudaError_t launch_pose(const LigView &L, const double *genes, int64_t P, int ngenes, float *out,
                        cudaStream_t st)
{
    int B;
    if (vdi::pick_block(L.n_atoms, &B)) return cudaErrorInvalidValue;
    if (P <= 0) return cudaSuccess;
    const size_t smem = sizeof(float) * 3 * (size_t)L.n_atoms * B;
    const int64_t blocks = (P + B - 1) / B;
    cudaError_t e;
    switch (B) {
    case 128:
        e = cudaFuncSetAttribute(pose_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) pose_kernel<128><<<(unsigned)blocks, 128, smem, st>>>(L, genes, P, ngenes, out);
        break;
    case 64:
        e = cudaFuncSetAttribute(pose_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) pose_kernel<64><<<(unsigned)blocks, 64, smem, st>>>(L, genes, P, ngenes, out);
        break;
    default:
        e = cudaFuncSetAttribute(pose_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) pose_kernel<32><<<(unsigned)blocks, 32, smem, st>>>(L, genes, P, ngenes, out);
    }
    if (e != cudaSuccess) return e;
    ++vdi::g_launches;
    return cudaGetLastError();
}

}  // namespace vd
