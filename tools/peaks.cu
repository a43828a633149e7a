// peaks.cu -- live B200 roofline denominators for bench.py (MEASURED_PEAKS.json
// carries only HBM copy and bf16 GEMM figures):
//   vdp_fp32_peak:  packed FFMA2 throughput (8 independent chains per thread)
//   vdp_l2_gather:  random 8-byte gathers from an L2-resident buffer
//   vdp_atom_gather: the score kernel's own per-atom gather pattern -- 4 LDG.64
//                    z-pair corners of a random type map + 2 LDG.256 elec/desolv
//                    bricks (96 B per atom) at uniformly random cells of
//                    same-size packed maps (context only: a pattern, not a ceiling)
//   vdp_l2_stream:   coalesced LDG.128 reads (L1-bypassing) of an L2-resident
//                    buffer by every SM: the hardware L2 read bandwidth ceiling
//   vdp_l2_sector:   random whole-sector (32-B, one LDG.256) reads of an
//                    L2-resident buffer: the L2 ceiling for scattered sectors
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void ffma2_kernel(float2 *out, int iters, float2 a, float2 b)
{
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-7f + k, k * 1e-3f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a, b);
    }
    float2 s = x[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) s = __fadd2_rn(s, x[k]);
    if (s.x == 12345.0f) out[threadIdx.x] = s;  // never true; keeps the chains live
}

__global__ void gather_kernel(const float2 *__restrict__ buf, uint64_t mask, int iters, float2 *out)
{
    uint64_t h = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
    float2 acc = make_float2(0.f, 0.f);
    for (int i = 0; i < iters; ++i) {
        float2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h ^= h << 13; h ^= h >> 7; h ^= h << 17;
            v[k] = __ldg(buf + (h & mask));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = __fadd2_rn(acc, v[k]);
    }
    if (acc.x == 12345.0f) out[0] = acc;
}

__device__ __forceinline__ void ld256(const float4 *p, float4 &lo, float4 &hi)
{
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z),
                   "=f"(hi.w)
                 : "l"(p));
}

__global__ void atom_gather_kernel(const float2 *__restrict__ zp, const float4 *__restrict__ ed,
                                   int n, int n_types, int iters, float *out)
{
    uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    const int nyz = n * n;
    const int64_t mstride = (int64_t)n * nyz;
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll 4
        for (int k = 0; k < 4; ++k) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            const int ix = (h >> 4) % (n - 1), iy = (h >> 12) % (n - 1), iz = (h >> 20) % (n - 1);
            const int m = h % n_types;
            const int idx = (ix * n + iy) * n + iz;
            const float2 *t = zp + mstride * m;
            const float2 a = __ldg(t + idx), b = __ldg(t + idx + n);
            const float2 c = __ldg(t + idx + nyz), d = __ldg(t + idx + nyz + n);
            float4 e0, d0, e1, d1;
            ld256(ed + 2 * (int64_t)idx, e0, d0);
            ld256(ed + 2 * (int64_t)(idx + nyz), e1, d1);
            acc += a.x + b.y + c.x + d.y + e0.x + d0.w + e1.y + d1.z;
        }
    }
    if (acc == 12345.0f) out[0] = acc;
}

__global__ void stream_kernel(const float4 *__restrict__ buf, int64_t n4, int passes, float *out)
{
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {
            const float4 a = __ldcg(buf + i), b = __ldcg(buf + i + stride);
            const float4 c = __ldcg(buf + i + 2 * stride), d = __ldcg(buf + i + 3 * stride);
            acc.x += a.x + b.y; acc.y += c.z + d.w; acc.z += a.w + c.x; acc.w += b.z + d.y;
        }
        for (; i < n4; i += stride) acc.x += __ldcg(buf + i).x;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.0f) out[0] = acc.x;
}

__global__ void sector_kernel(const float4 *__restrict__ buf, uint32_t mask, int iters, float *out)
{
    uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 777u;
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h ^= h << 13; h ^= h >> 17; h ^= h << 5;
            float4 lo, hi;
            asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y),
                           "=f"(hi.z), "=f"(hi.w)
                         : "l"(buf + 2 * (size_t)(h & mask)));
            acc += lo.x + hi.w;
        }
    }
    if (acc == 12345.0f) out[0] = acc;
}

static float time_it(void (*launch)(void *), void *arg)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(arg);  // warm
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / 5;
}

struct FArgs { float2 *out; int blocks, threads, iters; };
static void launch_ffma(void *p)
{
    FArgs *f = (FArgs *)p;
    ffma2_kernel<<<f->blocks, f->threads>>>(f->out, f->iters, make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f));
}
struct GArgs { const float2 *buf; uint64_t mask; float2 *out; int blocks, threads, iters; };
static void launch_gather(void *p)
{
    GArgs *g = (GArgs *)p;
    gather_kernel<<<g->blocks, g->threads>>>(g->buf, g->mask, g->iters, g->out);
}

extern "C" double vdp_fp32_peak_tflops(void)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    FArgs f;
    cudaMalloc(&f.out, 1024 * sizeof(float2));
    f.blocks = sms * 8;
    f.threads = 256;
    f.iters = 8192;
    const float ms = time_it(launch_ffma, &f);
    cudaFree(f.out);
    const double flops = (double)f.blocks * f.threads * f.iters * 8 * 2 /*lanes*/ * 2 /*fma*/;
    return flops / (ms * 1e-3) / 1e12;
}

extern "C" double vdp_l2_gather_gbs(int64_t bytes)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n = bytes / 8;  // power of two float2 elements
    GArgs g;
    cudaMalloc((void **)&g.buf, n * sizeof(float2));
    cudaMemset((void *)g.buf, 0, n * sizeof(float2));
    cudaMalloc(&g.out, sizeof(float2));
    g.mask = (uint64_t)n - 1;
    g.blocks = sms * 8;
    g.threads = 256;
    g.iters = 256;
    const float ms = time_it(launch_gather, &g);
    cudaFree((void *)g.buf);
    cudaFree(g.out);
    const double useful = (double)g.blocks * g.threads * g.iters * 8 * 8;  // bytes delivered
    return useful / (ms * 1e-3) / 1e9;
}

struct AArgs { const float2 *zp; const float4 *ed; int n, n_types, iters, blocks, threads; float *out; };
static void launch_atom(void *p)
{
    AArgs *a = (AArgs *)p;
    atom_gather_kernel<<<a->blocks, a->threads>>>(a->zp, a->ed, a->n, a->n_types, a->iters, a->out);
}

/* GB/s of 96-B atom gathers (the score kernel's inter pattern) over an n^3 grid
 * with n_types z-pair type maps plus one elec/desolv brick map. */
extern "C" double vdp_atom_gather_gbs(int n, int n_types)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t nodes = (size_t)n * n * n;
    AArgs a;
    cudaMalloc((void **)&a.zp, nodes * n_types * sizeof(float2));
    cudaMalloc((void **)&a.ed, nodes * 2 * sizeof(float4));
    cudaMemset((void *)a.zp, 0, nodes * n_types * sizeof(float2));
    cudaMemset((void *)a.ed, 0, nodes * 2 * sizeof(float4));
    cudaMalloc(&a.out, sizeof(float));
    a.n = n;
    a.n_types = n_types;
    a.blocks = sms * 16;
    a.threads = 128;
    a.iters = 128;
    const float ms = time_it(launch_atom, &a);
    cudaFree((void *)a.zp);
    cudaFree((void *)a.ed);
    cudaFree(a.out);
    const double atoms = (double)a.blocks * a.threads * a.iters * 4;
    return atoms * 96.0 / (ms * 1e-3) / 1e9;
}

struct SArgs { const float4 *buf; int64_t n4; int passes, blocks, threads; float *out; };
static void launch_stream(void *p)
{
    SArgs *a = (SArgs *)p;
    stream_kernel<<<a->blocks, a->threads>>>(a->buf, a->n4, a->passes, a->out);
}

/* GB/s of coalesced L2-resident reads (bytes <= ~1/3 of L2 keeps it resident on both dies) */
extern "C" double vdp_l2_stream_gbs(int64_t bytes)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    SArgs a;
    a.n4 = bytes / 16;
    cudaMalloc((void **)&a.buf, a.n4 * sizeof(float4));
    cudaMemset((void *)a.buf, 0, a.n4 * sizeof(float4));
    cudaMalloc(&a.out, sizeof(float));
    a.blocks = sms * 4;
    a.threads = 512;
    a.passes = 16;
    const float ms = time_it(launch_stream, &a);
    cudaFree((void *)a.buf);
    cudaFree(a.out);
    return (double)a.n4 * 16.0 * a.passes / (ms * 1e-3) / 1e9;
}

struct QArgs { const float4 *buf; uint32_t mask; int iters, blocks, threads; float *out; };
static void launch_sector(void *p)
{
    QArgs *a = (QArgs *)p;
    sector_kernel<<<a->blocks, a->threads>>>(a->buf, a->mask, a->iters, a->out);
}

/* GB/s of random 32-B sector reads from an L2-resident buffer (bytes: power of two) */
extern "C" double vdp_l2_sector_gbs(int64_t bytes)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    QArgs a;
    const int64_t sectors = bytes / 32;
    cudaMalloc((void **)&a.buf, sectors * 32);
    cudaMemset((void *)a.buf, 0, sectors * 32);
    cudaMalloc(&a.out, sizeof(float));
    a.mask = (uint32_t)(sectors - 1);
    a.blocks = sms * 8;
    a.threads = 256;
    a.iters = 128;
    const float ms = time_it(launch_sector, &a);
    cudaFree((void *)a.buf);
    cudaFree(a.out);
    return (double)a.blocks * a.threads * a.iters * 8 * 32.0 / (ms * 1e-3) / 1e9;
}
