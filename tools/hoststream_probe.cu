// Csr SpMV with both operands in pinned host memory, as ONE cooperative kernel.
//
// The reference's apply on host arrays (LinOp.apply, src/base.py:60-70, with
// the executor migration of src/base.py:99-127) is transfer-bound on a GPU:
// b goes up and x comes down over PCIe, and the SpMV itself is a third of the
// link time. Copy-engine pipelining (chunked cudaMemcpyAsync + events) pays a
// per-chunk cost when both directions are busy (tools/e2e_probe.py: 8 chunks
// each way = 435 us vs 341 us for one copy each way on C2), so the chunk
// count cannot go up far enough to hide the fill and drain.
//
// Here the streaming is done by the SMs, at cache-line granularity:
//   * producer CTAs (the first `nprod`) read b from the mapped host buffer in
//     64 KB chunks (16-byte loads, 16 in flight per thread), write it to a
//     device staging copy and publish each chunk with a release flag
//     (flags[c] = epoch; epochs make the flags reusable without a reset);
//   * consumer CTAs take row tiles in increasing order, wait (one thread,
//     acquire loads) until every b chunk the tile's columns reach has landed
//     (tile_need[t], planned once per matrix), reduce the tile's rows with the
//     classical sub-warp scheme (same order of operations as
//     csr_classical_kernel, so the results are identical), stage them in
//     shared memory and store them straight into the host x with coalesced
//     16-byte stores (posted PCIe writes).
// So H2D, SpMV and D2H overlap at tile granularity with no per-chunk API cost.
// The cooperative launch guarantees every CTA is resident, so consumers that
// spin on flags can never starve the producers.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "common.cuh"

namespace b200sp {

constexpr int HS_BLOCK = 256;
constexpr int HS_CHUNK_BYTES = 64 * 1024;
constexpr int HS_MAX_TILE_BYTES = 32 * 1024;

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T, int SW, int U>
__global__ void __launch_bounds__(HS_BLOCK)
csr_host_stream_kernel(int64_t n, int64_t ncols, const int* __restrict__ rp, const int* __restrict__ ci,
                       const T* __restrict__ v, const T* bh, T* bd, T* xh, const int* __restrict__ tile_need,
                       int tile_rows, int* flags, int epoch, int nprod, int vec) {
    extern __shared__ __align__(16) unsigned char hs_smem[];
    constexpr int64_t CHUNK = HS_CHUNK_BYTES / sizeof(T);
    const int64_t nchunks = (ncols + CHUNK - 1) / CHUNK;
    if ((int)blockIdx.x < nprod) {
        // ---- producer: host b -> device staging, chunk by chunk ----
        constexpr int NV = HS_CHUNK_BYTES / 16 / HS_BLOCK;
        for (int64_t c = blockIdx.x; c < nchunks; c += nprod) {
            const int64_t e0 = c * CHUNK, e1 = min(e0 + CHUNK, ncols);
            if (vec && e1 - e0 == CHUNK) {
                const int4* src = reinterpret_cast<const int4*>(bh + e0);
                int4* dst = reinterpret_cast<int4*>(bd + e0);
                int4 r[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) r[i] = src[threadIdx.x + i * HS_BLOCK];
#pragma unroll
                for (int i = 0; i < NV; ++i) dst[threadIdx.x + i * HS_BLOCK] = r[i];
            } else {
                for (int64_t e = e0 + threadIdx.x; e < e1; e += HS_BLOCK) bd[e] = bh[e];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                st_release_gpu(flags + c, epoch);
            }
        }
        return;
    }
    // ---- consumers: row tiles in increasing order ----
    T* xs = reinterpret_cast<T*>(hs_smem);
    const int ncons = gridDim.x - nprod;
    const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
    const int lane = threadIdx.x & (SW - 1);
    constexpr int NSW = HS_BLOCK / SW;
    int ready = 0;  // thread 0: chunks [0, ready) have landed
    for (int64_t t = (int)blockIdx.x - nprod; t < ntiles; t += ncons) {
        const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
        if (threadIdx.x == 0) {
            const int need = tile_need[t];
            while (ready <= need) {
                if (ld_acquire_gpu(flags + ready) == epoch)
                    ++ready;
                else
                    __nanosleep(100);
            }
        }
        __syncthreads();
        const int64_t wfirst = r0 + (int64_t)(threadIdx.x / 32) * (32 / SW) * U;
        for (int64_t row0 = r0 + (int64_t)(threadIdx.x / SW) * U, w0 = wfirst; w0 < r1;
             row0 += NSW * U, w0 += NSW * U) {
            int s[U], len[U];
            int ptr_next = row0 < r1 ? __ldg(rp + row0) : 0;
            int maxlen = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                s[u] = ptr_next;
                ptr_next = (row0 + u < r1) ? __ldg(rp + row0 + u + 1) : ptr_next;
                len[u] = ptr_next - s[u];
                maxlen = max(maxlen, len[u]);
            }
            T acc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = 0;
            for (int k = lane; k < maxlen; k += SW) {
                int c[U];
                T vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool ok = k < len[u];
                    c[u] = ok ? __ldg(ci + s[u] + k) : -1;
                    vv[u] = ok ? __ldg(v + s[u] + k) : T(0);
                }
                // b was written during this kernel: coherent L2 loads only
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (c[u] >= 0) acc[u] += vv[u] * __ldcg(bd + c[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = subwarp_sum<SW>(acc[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u % SW == lane && row0 + u < r1) xs[row0 + u - r0] = acc[u];
        }
        __syncthreads();
        const int cnt = (int)(r1 - r0);
        T* dst = xh + r0;
        constexpr int PER = 16 / sizeof(T);
        if (vec && cnt % PER == 0) {
            const int4* s4 = reinterpret_cast<const int4*>(xs);
            int4* d4 = reinterpret_cast<int4*>(dst);
            for (int i = threadIdx.x; i < cnt / PER; i += HS_BLOCK) d4[i] = s4[i];
        } else {
            for (int i = threadIdx.x; i < cnt; i += HS_BLOCK) dst[i] = xs[i];
        }
        __syncthreads();
    }
}

// tile_need[t] = index of the last b chunk the columns of row tile t reach (-1: empty tile)
__global__ void __launch_bounds__(256)
csr_tile_chunks_kernel(int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, int tile_rows,
                       int64_t chunk_elems, int* __restrict__ need) {
    __shared__ int sh[8];
    const int64_t t = blockIdx.x;
    const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
    const int e0 = rp[r0], e1 = rp[r1];
    int m = -1;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) m = max(m, ci[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        int r = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = max(r, sh[w]);
        need[t] = r < 0 ? -1 : (int)(r / chunk_elems);
    }
}

template <typename T, int SW>
static int launch_host_stream(int64_t n, int64_t ncols, const int* rp, const int* ci, const T* v, const T* bh,
                              T* bd, T* xh, const int* need, int tile_rows, int* flags, int epoch, cudaStream_t st) {
    constexpr int U = ClassicalRows<SW>::v;
    auto kern = csr_host_stream_kernel<T, SW, U>;
    const size_t smem = (size_t)tile_rows * sizeof(T);
    int per_sm = 0;
    B200SP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, HS_BLOCK, smem));
    B200SP_REQUIRE(per_sm > 0, B200SP_ECUDA, "csr host stream: kernel cannot be resident");
    per_sm = std::min(per_sm, tuning("hs_per_sm", 3));
    const int grid = per_sm * kNumSMs;
    int nprod = tuning("hs_producers", 4);  // fewer readers measured faster: 4 -> 537 us, 32 -> 661 us on C2
    nprod = std::max(1, std::min(nprod, grid / 2));
    const int vec = aligned16(bh) && aligned16(bd) && aligned16(xh);
    void* args[] = {(void*)&n, (void*)&ncols, (void*)&rp, (void*)&ci, (void*)&v, (void*)&bh, (void*)&bd,
                    (void*)&xh, (void*)&need, (void*)&tile_rows, (void*)&flags, (void*)&epoch, (void*)&nprod,
                    (void*)&vec};
    B200SP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(HS_BLOCK), args,
                                                  smem, st));
    return B200SP_OK;
}

template <typename T>
static int csr_host_stream(int64_t n, int64_t ncols, const int* rp, const int* ci, const T* v, const T* b_host,
                           T* b_dev, T* x_host, const int* tile_need, int tile_rows, int* flags, int epoch,
                           int subwarp, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(tile_rows > 0 && tile_rows % 4 == 0 && (size_t)tile_rows * sizeof(T) <= HS_MAX_TILE_BYTES,
                   B200SP_EINVAL, "csr host stream: tile_rows must be a multiple of 4 with <= %d bytes of x (got %d)",
                   HS_MAX_TILE_BYTES, tile_rows);
    B200SP_REQUIRE(epoch > 0, B200SP_EINVAL, "csr host stream: epoch must be positive (got %d)", epoch);
    // the host buffers must be page-locked and mapped (UVA): translate them
    void* bdev = nullptr;
    void* xdev = nullptr;
    if (cudaHostGetDevicePointer(&bdev, const_cast<T*>(b_host), 0) != cudaSuccess ||
        cudaHostGetDevicePointer(&xdev, x_host, 0) != cudaSuccess) {
        cudaGetLastError();
        set_error("csr host stream: b and x must be pinned host memory (cudaHostAlloc / pin_memory)");
        return B200SP_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    const T* bh = static_cast<const T*>(bdev);
    T* xh = static_cast<T*>(xdev);
    int rc;
    switch (subwarp) {
        case 1: rc = launch_host_stream<T, 1>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        case 2: rc = launch_host_stream<T, 2>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        case 4: rc = launch_host_stream<T, 4>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        case 8: rc = launch_host_stream<T, 8>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        case 16: rc = launch_host_stream<T, 16>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        case 32: rc = launch_host_stream<T, 32>(n, ncols, rp, ci, v, bh, b_dev, xh, tile_need, tile_rows, flags, epoch, st); break;
        default: set_error("csr host stream: subwarp must be a power of two <= 32 (got %d)", subwarp);
                 return B200SP_EINVAL;
    }
    if (rc != B200SP_OK) return rc;
    count_launch();
    return check_launch("csr_host_stream");
}

}  // namespace b200sp

using namespace b200sp;

extern "C" {

int32_t b200sp_csr_host_chunk_elems(int32_t value_bytes) {
    return value_bytes == 4 || value_bytes == 8 ? HS_CHUNK_BYTES / value_bytes : -1;
}

int b200sp_csr_tile_chunks(int64_t n, const int32_t* rp, const int32_t* ci, int32_t tile_rows, int64_t chunk_elems,
                           int32_t* need, void* stream) {
    if (n == 0) return B200SP_OK;
    B200SP_REQUIRE(tile_rows > 0 && chunk_elems > 0, B200SP_EINVAL, "csr tile chunks: bad tile_rows / chunk_elems");
    const int64_t ntiles = ceil_div(n, tile_rows);
    csr_tile_chunks_kernel<<<(unsigned)ntiles, 256, 0, as_stream(stream)>>>(n, rp, ci, tile_rows, chunk_elems, need);
    count_launch();
    return check_launch("csr_tile_chunks");
}

int b200sp_csr_spmv_host_f64(int64_t n, int64_t ncols, const int32_t* rp, const int32_t* ci, const double* v,
                             const double* b_host, double* b_dev, double* x_host, const int32_t* tile_need,
                             int32_t tile_rows, int32_t* flags, int32_t epoch, int32_t subwarp, void* stream) {
    return csr_host_stream<double>(n, ncols, rp, ci, v, b_host, b_dev, x_host, tile_need, tile_rows, flags, epoch,
                                   subwarp, stream);
}

int b200sp_csr_spmv_host_f32(int64_t n, int64_t ncols, const int32_t* rp, const int32_t* ci, const float* v,
                             const float* b_host, float* b_dev, float* x_host, const int32_t* tile_need,
                             int32_t tile_rows, int32_t* flags, int32_t epoch, int32_t subwarp, void* stream) {
    return csr_host_stream<float>(n, ncols, rp, ci, v, b_host, b_dev, x_host, tile_need, tile_rows, flags, epoch,
                                  subwarp, stream);
}

}  // extern "C"
