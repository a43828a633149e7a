/*
 * vd_mugd.cu -- MUGD grid files straight into a device grid.
 *
 * Format (vd/grids.py:232-258 write_grid_set, :269-303 read_grid_set; pinned by
 * pkg/tests/test_grids.py:206-272): 'MUGD' | u32 version (1) | u32 nx, ny, nz |
 * f32 origin[3] | f32 spacing | u32 map_count | per map: u16 label length, UTF-8
 * label, nx*ny*nz f32 little-endian payload, x fastest.  Nothing may follow the
 * last payload.
 *
 * The reference reads each payload into a numpy array and transposes it on the host
 * into the z-fastest C order the kernels index.  Here the payload bytes go from the
 * file into pinned host staging (two buffers, so reading map m+1 overlaps map m's
 * copy), are copied to the device as they are, and a tiled shared-memory transpose
 * writes them into the grid's (n_maps, nx, ny, nz) stack, counting non-finite values
 * on the way (the reference's GridMapSet check, vd/grids.py:95-105).  No host-side
 * transpose, no pageable copy.
 */
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "vd_internal.h"

namespace {

struct FileCloser {
    FILE *f;
    ~FileCloser()
    {
        if (f) fclose(f);
    }
};

/* 0 ok, -2 format error (message set) */
int read_exact(FILE *f, void *dst, size_t n, const char *what)
{
    if (fread(dst, 1, n, f) != n) {
        vdi::set_error(std::string("unexpected end of MUGD stream while reading ") + what);
        return -2;
    }
    return 0;
}

struct Header {
    uint32_t nx, ny, nz, count;
    float origin[3], spacing;
    std::vector<std::string> labels;
    std::vector<long> payload_at;
};

int parse(FILE *f, Header &h)
{
    fseek(f, 0, SEEK_END);
    const long size = ftell(f);
    fseek(f, 0, SEEK_SET);
    char magic[4];
    if (int rc = read_exact(f, magic, 4, "magic")) return rc;
    if (memcmp(magic, "MUGD", 4) != 0) {
        vdi::set_error("bad magic, expected b'MUGD'");
        return -2;
    }
    uint32_t version;
    if (int rc = read_exact(f, &version, 4, "version")) return rc;
    if (version != 1) {
        vdi::set_error("unsupported MUGD version " + std::to_string(version) + ", expected 1");
        return -2;
    }
    uint32_t dims[3];
    if (int rc = read_exact(f, dims, 12, "dims")) return rc;
    if (int rc = read_exact(f, h.origin, 12, "origin")) return rc;
    if (int rc = read_exact(f, &h.spacing, 4, "spacing")) return rc;
    if (int rc = read_exact(f, &h.count, 4, "map count")) return rc;
    h.nx = dims[0]; h.ny = dims[1]; h.nz = dims[2];
    const uint64_t payload = 4ull * h.nx * h.ny * h.nz;
    for (uint32_t m = 0; m < h.count; ++m) {
        uint16_t len;
        if (int rc = read_exact(f, &len, 2, "label length")) return rc;
        std::string label(len, '\0');
        if (int rc = read_exact(f, label.data(), len, "label")) return rc;
        h.labels.push_back(label);
        const long at = ftell(f);
        h.payload_at.push_back(at);
        /* skip the payload, checking it is all there */
        if ((uint64_t)(size - at) < payload || fseek(f, (long)payload, SEEK_CUR) != 0) {
            vdi::set_error("unexpected end of MUGD stream while reading payload of map '" + label + "'");
            return -2;
        }
    }
    if (size > ftell(f)) {
        vdi::set_error("trailing bytes after final map payload (size mismatch)");
        return -2;
    }
    return 0;
}

/* (z, x) plane of row y, x fastest  ->  C order (x, y, z), z fastest; 32 x 32 tiles */
__global__ void xfast_to_c_kernel(const float *__restrict__ src, float *__restrict__ dst, int nx,
                                  int ny, int nz, int *nonfinite)
{
    __shared__ float tile[32][33];
    const int y = blockIdx.z;
    const int x0 = blockIdx.x * 32, z0 = blockIdx.y * 32;
    int bad = 0;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {  /* read: x fastest (coalesced) */
        const int z = z0 + k, x = x0 + threadIdx.x;
        if (z < nz && x < nx) {
            const float v = src[((int64_t)z * ny + y) * nx + x];
            bad |= !isfinite(v);
            tile[k][threadIdx.x] = v;
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {  /* write: z fastest (coalesced) */
        const int x = x0 + k, z = z0 + threadIdx.x;
        if (x < nx && z < nz) dst[((int64_t)x * ny + y) * nz + z] = tile[threadIdx.x][k];
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

}  // namespace

extern "C" {

int vd_mugd_read_header(const char *path, vd_mugd_info *info, char *labels, int labels_cap)
{
    FileCloser fc{fopen(path, "rb")};
    if (!fc.f) {
        vdi::set_error(std::string("cannot open MUGD file ") + path);
        return -1;
    }
    Header h;
    if (int rc = parse(fc.f, h)) return rc;
    info->n_maps = (int32_t)h.count;
    info->nx = (int32_t)h.nx; info->ny = (int32_t)h.ny; info->nz = (int32_t)h.nz;
    for (int k = 0; k < 3; ++k) info->origin[k] = h.origin[k];
    info->spacing = h.spacing;
    int need = 0;
    for (auto &l : h.labels) need += (int)l.size() + 1;
    info->labels_bytes = need;
    if (labels) {
        if (labels_cap < need) {
            vdi::set_error("vd_mugd_read_header: label buffer too small");
            return -1;
        }
        int off = 0;
        for (auto &l : h.labels) {
            memcpy(labels + off, l.data(), l.size());
            labels[off + l.size()] = '\0';
            off += (int)l.size() + 1;
        }
    }
    return 0;
}

int vd_grid_load_mugd(const char *path, vd_grid **out)
{
    *out = nullptr;
    FileCloser fc{fopen(path, "rb")};
    if (!fc.f) {
        vdi::set_error(std::string("cannot open MUGD file ") + path);
        return -1;
    }
    Header h;
    if (int rc = parse(fc.f, h)) return rc;
    if (h.count < 1 || h.nx < 2 || h.ny < 2 || h.nz < 2 || !(h.spacing > 0.f)) {
        vdi::set_error("vd_grid_load_mugd: bad grid shape in MUGD header");
        return -2;
    }
    const size_t nodes = (size_t)h.nx * h.ny * h.nz;
    float lo[3], hi[3];
    const uint32_t d[3] = {h.nx, h.ny, h.nz};
    for (int k = 0; k < 3; ++k) {  /* GridSpec.upper = origin + (n - 1) * spacing, in f64 */
        lo[k] = h.origin[k];
        hi[k] = (float)((double)h.origin[k] + (double)(d[k] - 1) * (double)h.spacing);
    }
    vd_grid *g = nullptr;
    if (vd_grid_create(nullptr, (int)h.count, (int)h.nx, (int)h.ny, (int)h.nz, lo, hi, h.spacing, &g))
        return -1;
    float *pin[2] = {nullptr, nullptr}, *dev[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int *d_bad = nullptr;
    cudaStream_t st = nullptr;
    int rc = 0;
    auto ck = [&](cudaError_t e, const char *what) {
        if (rc == 0 && !vdi::check(e, what)) rc = -1;
        return rc == 0;
    };
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    for (int b = 0; b < 2 && rc == 0; ++b) {
        ck(cudaHostAlloc((void **)&pin[b], nodes * sizeof(float), cudaHostAllocDefault), "pinned staging");
        ck(cudaMalloc((void **)&dev[b], nodes * sizeof(float)), "device staging");
        ck(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming), "event");
    }
    ck(cudaMalloc((void **)&d_bad, sizeof(int) * h.count), "flags");
    ck(cudaMemsetAsync(d_bad, 0, sizeof(int) * h.count, st), "flags");
    const dim3 blk(32, 8), grd((h.nx + 31) / 32, (h.nz + 31) / 32, h.ny);
    for (uint32_t m = 0; m < h.count && rc == 0; ++m) {
        const int b = (int)(m & 1);
        /* staging buffer b is free once map m-2's copy has drained it */
        if (m >= 2) ck(cudaEventSynchronize(done[b]), "staging reuse");
        if (rc) break;
        fseek(fc.f, h.payload_at[m], SEEK_SET);
        if (fread(pin[b], sizeof(float), nodes, fc.f) != nodes) {
            vdi::set_error("unexpected end of MUGD stream while reading payload of map '" + h.labels[m] + "'");
            rc = -2;
            break;
        }
        ck(cudaMemcpyAsync(dev[b], pin[b], nodes * sizeof(float), cudaMemcpyHostToDevice, st), "H2D payload");
        ck(cudaEventRecord(done[b], st), "event");
        if (rc) break;
        xfast_to_c_kernel<<<grd, blk, 0, st>>>(dev[b], g->d_maps + nodes * m, (int)h.nx, (int)h.ny,
                                               (int)h.nz, d_bad + m);
        ++vdi::g_launches;
        ck(cudaGetLastError(), "transpose kernel");
    }
    std::vector<int> bad(h.count, 0);
    if (rc == 0) ck(cudaMemcpyAsync(bad.data(), d_bad, sizeof(int) * h.count, cudaMemcpyDeviceToHost, st), "flags");
    if (rc == 0) ck(cudaStreamSynchronize(st), "sync");
    for (uint32_t m = 0; m < h.count && rc == 0; ++m)
        if (bad[m]) {
            vdi::set_error("map '" + h.labels[m] + "' contains non-finite values");
            rc = -2;
        }
    if (st) cudaStreamSynchronize(st);
    for (int b = 0; b < 2; ++b) {
        if (pin[b]) cudaFreeHost(pin[b]);
        if (dev[b]) cudaFree(dev[b]);
        if (done[b]) cudaEventDestroy(done[b]);
    }
    if (d_bad) cudaFree(d_bad);
    if (st) cudaStreamDestroy(st);
    if (rc == 0 && !vdi::make_packed(g)) rc = -1;
    if (rc) {
        vd_grid_destroy(g);
        return rc;
    }
    *out = g;
    return 0;
}

}  // extern "C"
