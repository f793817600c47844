// Device-side assembly of coordinate triples: the
// reference's MatrixData.canonicalize (src/formats.py:40-53) restated on the
// GPU, bit for bit:
//   * order = np.lexsort((cols, rows)) -- a STABLE sort by (row, col); here a
//     stable LSD radix sort of the composite key row * ncols + col (8-bit
//     digits, as many passes as the key has bits) carrying the original
//     position;
//   * duplicates: if ANY coordinate repeats, every group is summed with
//     np.add.at into zeros, i.e. 0.0 + v_1 + v_2 + ... in input order (so a
//     lone -0.0 becomes +0.0); with no duplicate at all the values pass
//     through unchanged. Each group is summed sequentially by one thread.
// Radix pass = per-tile digit histogram -> one exclusive scan over
// (digit, tile) -> stable scatter: inside a tile, items are ranked warp by
// warp with __match_any_sync, so equal digits keep their input order.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "common.cuh"

namespace b200sp {

constexpr int RS_BLOCK = 256;
constexpr int RS_ITEMS = 16;                       // keys per thread per pass
constexpr int RS_TILE = RS_BLOCK * RS_ITEMS;       // 4096 keys per tile
constexpr int RS_WARPS = RS_BLOCK / 32;
constexpr int RS_BINS = 256;

// item j of warp w in tile t sits at t*TILE + w*(32*ITEMS) + k*32 + lane
__device__ __forceinline__ int64_t rs_index(int64_t tile, int w, int k, int lane) {
    return tile * RS_TILE + (int64_t)w * (32 * RS_ITEMS) + k * 32 + lane;
}

__global__ void __launch_bounds__(RS_BLOCK)
rs_hist_kernel(int64_t count, const uint64_t* __restrict__ keys, int shift, int ntiles, int* __restrict__ counts) {
    __shared__ int h[RS_BINS];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 4
    for (int k = 0; k < RS_ITEMS; ++k) {
        const int64_t i = rs_index(blockIdx.x, w, k, lane);
        if (i < count) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(RS_BLOCK)
rs_scatter_kernel(int64_t count, const uint64_t* __restrict__ keys, const int* __restrict__ perm, int shift,
                  int ntiles, const int* __restrict__ offs, uint64_t* __restrict__ keys_out, int* __restrict__ perm_out) {
    __shared__ int wcnt[RS_WARPS][RS_BINS];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = threadIdx.x; d < RS_WARPS * RS_BINS; d += RS_BLOCK) (&wcnt[0][0])[d] = 0;
    __syncthreads();
    int dig[RS_ITEMS], rank[RS_ITEMS];
    uint64_t kv[RS_ITEMS];
    int pv[RS_ITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < RS_ITEMS; ++k) {
        const int64_t i = rs_index(blockIdx.x, w, k, lane);
        const bool ok = i < count;
        kv[k] = ok ? keys[i] : 0;
        pv[k] = ok ? perm[i] : 0;
        const int d = ok ? (int)((kv[k] >> shift) & 0xff) : RS_BINS;  // RS_BINS: no item
        dig[k] = d;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int before = __popc(peers & lt);
        const int base = d < RS_BINS ? wcnt[w][d] : 0;
        rank[k] = base + before;
        __syncwarp();
        if (d < RS_BINS && before == 0) wcnt[w][d] = base + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps, per digit (thread t owns digit t)
    {
        const int d = threadIdx.x;
        int run = 0;
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            const int c = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RS_ITEMS; ++k) {
        const int d = dig[k];
        if (d < RS_BINS) {
            const int64_t pos = (int64_t)offs[(int64_t)d * ntiles + blockIdx.x] + wcnt[w][d] + rank[k];
            keys_out[pos] = kv[k];
            perm_out[pos] = pv[k];
        }
    }
}

__global__ void rs_keys_kernel(int64_t count, const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                               int64_t ncols, uint64_t* __restrict__ keys, int* __restrict__ perm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint64_t)rows[i] * (uint64_t)ncols + (uint64_t)cols[i];
        perm[i] = (int)i;
    }
}

// heads[i] = 1 where a new coordinate starts
__global__ void rs_heads_kernel(int64_t count, const uint64_t* __restrict__ keys, int* __restrict__ heads) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per group: decode (row, col), sum the group's values in input
// order starting from +0.0 when the matrix has duplicates (np.add.at into
// np.zeros), else copy the single value through
template <typename T>
__global__ void rs_groups_kernel(int64_t count, const uint64_t* __restrict__ keys, const int* __restrict__ perm,
                                 const int* __restrict__ heads, const int* __restrict__ gid, const double* __restrict__ vals,
                                 int64_t ncols, int* __restrict__ rows_out, int* __restrict__ cols_out,
                                 T* __restrict__ vals_out) {
    const int64_t ngroups = gid[count];
    const bool dups = ngroups < count;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        if (!heads[i]) continue;
        const uint64_t key = keys[i];
        double s = vals[perm[i]];
        if (dups) {
            s = 0.0 + s;
            for (int64_t j = i + 1; j < count && keys[j] == key; ++j) s = s + vals[perm[j]];
        }
        const int64_t g = gid[i];
        rows_out[g] = (int)(key / (uint64_t)ncols);
        cols_out[g] = (int)(key % (uint64_t)ncols);
        vals_out[g] = (T)s;
    }
}

}  // namespace b200sp

using namespace b200sp;

extern "C" {

int b200sp_exclusive_scan_i32(int64_t count, const int32_t* in, int32_t* out, long long* ws, void* stream);
int64_t b200sp_scan_workspace_elems(int64_t count);

/* workspace bytes of b200sp_assemble_coo for `count` triples */
int64_t b200sp_assemble_workspace_bytes(int64_t count) {
    const int64_t ntiles = ceil_div(count, RS_TILE);
    const int64_t nc = (int64_t)RS_BINS * ntiles;
    const int64_t scan_n = std::max<int64_t>(nc, count) + 1;
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    return al(2 * count * 8) + al(2 * count * 4) + al(2 * (nc + 1) * 4) + al(2 * (count + 1) * 4) +
           al(b200sp_scan_workspace_elems(scan_n) * 8);
}

#define ASSEMBLE_T(T, SUF)                                                                                       \
    int b200sp_assemble_coo_##SUF(int64_t count, const int64_t* rows, const int64_t* cols, const double* vals,    \
                                  int64_t nrows, int64_t ncols, int32_t* rows_out, int32_t* cols_out, T* vals_out, \
                                  int32_t* nnz_out, void* ws, void* stream) {                                     \
        return assemble<T>(count, rows, cols, vals, nrows, ncols, rows_out, cols_out, vals_out, nnz_out, ws, stream); \
    }

}  // extern "C"

namespace b200sp {
template <typename T>
static int assemble(int64_t count, const int64_t* rows, const int64_t* cols, const double* vals, int64_t nrows,
                    int64_t ncols, int32_t* rows_out, int32_t* cols_out, T* vals_out, int32_t* nnz_out, void* ws,
                    void* stream) {
    cudaStream_t st = as_stream(stream);
    B200SP_REQUIRE(count < INT_MAX, B200SP_EUNSUPPORTED, "assemble: more than 2^31-1 triples");
    B200SP_REQUIRE(nrows >= 0 && ncols >= 0 && nrows < INT_MAX && ncols < INT_MAX, B200SP_EUNSUPPORTED,
                   "assemble: dimensions must fit int32");
    if (count == 0) {
        B200SP_CHECK_CUDA(cudaMemsetAsync(nnz_out, 0, sizeof(int32_t), st));
        return B200SP_OK;
    }
    const int64_t ntiles = ceil_div(count, RS_TILE);
    const int64_t nc = (int64_t)RS_BINS * ntiles;
    const int64_t scan_n = std::max<int64_t>(nc, count) + 1;
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    char* p = (char*)ws;
    uint64_t* k0 = (uint64_t*)p;
    uint64_t* k1 = k0 + count;
    p += al(2 * count * 8);
    int* p0 = (int*)p;
    int* p1 = p0 + count;
    p += al(2 * count * 4);
    int* cnt = (int*)p;
    int* off = cnt + nc + 1;
    p += al(2 * (nc + 1) * 4);
    int* heads = (int*)p;
    int* gid = heads + count + 1;
    p += al(2 * (count + 1) * 4);
    long long* sws = (long long*)p;
    const int g = grid_for(count, 256, 8);
    rs_keys_kernel<<<g, 256, 0, st>>>(count, rows, cols, ncols, k0, p0);
    const uint64_t maxkey = (uint64_t)std::max<int64_t>(nrows, 1) * (uint64_t)std::max<int64_t>(ncols, 1) - 1;
    int bits = 0;
    while (bits < 64 && (maxkey >> bits)) ++bits;
    int passes = 0;
    for (int shift = 0; shift < bits; shift += 8, ++passes) {
        rs_hist_kernel<<<(unsigned)ntiles, RS_BLOCK, 0, st>>>(count, k0, shift, (int)ntiles, cnt);
        int rc = b200sp_exclusive_scan_i32(nc, cnt, off, sws, stream);
        if (rc != B200SP_OK) return rc;
        rs_scatter_kernel<<<(unsigned)ntiles, RS_BLOCK, 0, st>>>(count, k0, p0, shift, (int)ntiles, off, k1, p1);
        std::swap(k0, k1);
        std::swap(p0, p1);
        count_launch(2);
    }
    rs_heads_kernel<<<g, 256, 0, st>>>(count, k0, heads);
    int rc = b200sp_exclusive_scan_i32(count, heads, gid, sws, stream);
    if (rc != B200SP_OK) return rc;
    rs_groups_kernel<T><<<g, 256, 0, st>>>(count, k0, p0, heads, gid, vals, ncols, rows_out, cols_out, vals_out);
    B200SP_CHECK_CUDA(cudaMemcpyAsync(nnz_out, gid + count, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    count_launch(3);
    return check_launch("assemble_coo");
}
}  // namespace b200sp

extern "C" {
ASSEMBLE_T(double, f64)
ASSEMBLE_T(float, f32)
}
