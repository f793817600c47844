// Read-bandwidth of HBM streaming patterns (B200): does chunk-per-CTA
// streaming (load-balanced CSR tiles, Coo warp chunks) lose to grid-stride
// streaming at the same bytes?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/spp tools/stream_pattern_probe.cu && /tmp/spp
//
// Each kernel sums 1 GiB of doubles with 128-bit loads, 256-thread CTAs:
//   gridstride  : CTA-sized 4 KiB blocks dealt round-robin over a 2-wave grid
//   chunk/CTA   : each CTA (one per chunk, many waves) walks its own contiguous
//                 chunk of `chunk` bytes, the CTA's threads side by side
//   chunk/warp  : each warp walks its own contiguous chunk
#include <cstdio>
#include <cstdint>

__device__ double g_sink;
__device__ __forceinline__ double sum_of(float v) { return v; }
__device__ __forceinline__ double sum_of(double v) { return v; }
__device__ __forceinline__ double sum_of(double2 v) { return v.x + v.y; }
__device__ __forceinline__ double sum_of(float4 v) { return (double)v.x + v.y + v.z + v.w; }

__global__ void k_gridstride(const double2* __restrict__ a, int64_t n2) {
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) g_sink = s;
}

__global__ void k_chunk_cta(const double2* __restrict__ a, int64_t n2, int64_t per) {
    double s = 0;
    const int64_t base = (int64_t)blockIdx.x * per;
    for (int64_t i = base + threadIdx.x; i < base + per && i < n2; i += blockDim.x) {
        double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) g_sink = s;
}

__global__ void k_chunk_warp(const double2* __restrict__ a, int64_t n2, int64_t per) {
    double s = 0;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t base = w * per;
    for (int64_t i = base + lane; i < base + per && i < n2; i += 32) {
        double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) g_sink = s;
}

// element width / cache policy: T = float, double, double2; POL 0 = __ldcs
// (evict-first streaming), 1 = __ldg (L1-allocating), 2 = plain load
template <typename T, int POL>
__global__ void k_width(const T* __restrict__ a, int64_t n) {
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T v = POL == 0 ? __ldcs(a + i) : POL == 1 ? __ldg(a + i) : a[i];
        s += sum_of(v);
    }
    if (s == 12345.678) g_sink = s;
}

// SpMV-like streams: n entries of (int32 column, double value) read as two
// arrays (1/3 + 2/3 of the bytes) with VEC entries per lane per load
// (VEC 1: 4-byte + 8-byte loads, VEC 4: int4 + 2x double2), optionally a
// gather b[col] per entry (b = 2M doubles, L2-resident, 27-point-like columns)
// and one 8-byte store per 27 entries (the x write)
template <int VEC, bool GATHER, bool WRITE>
__global__ void k_spmv_like(const int* __restrict__ ci, const double* __restrict__ v, const double* __restrict__ b,
                            double* __restrict__ x, int64_t n) {
    double s = 0;
    const int64_t nv = n / VEC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        if (VEC == 1) {
            const int c = __ldg(ci + i);
            const double a = __ldg(v + i);
            s += GATHER ? a * __ldg(b + c) : a + c;
        } else {
            const int4 c = __ldg(reinterpret_cast<const int4*>(ci) + i);
            const double2 a0 = __ldg(reinterpret_cast<const double2*>(v) + 2 * i);
            const double2 a1 = __ldg(reinterpret_cast<const double2*>(v) + 2 * i + 1);
            if (GATHER)
                s += a0.x * __ldg(b + c.x) + a0.y * __ldg(b + c.y) + a1.x * __ldg(b + c.z) + a1.y * __ldg(b + c.w);
            else
                s += a0.x + a0.y + a1.x + a1.y + c.x + c.y + c.z + c.w;
        }
        if (WRITE && (i % (27 / VEC)) == 0) x[(i / (27 / VEC)) % 2097152] = s;
    }
    if (s == 12345.678) g_sink = s;
}

// Ell-like SpMV (27 entries per row, column-major ci / v, thread per row,
// grid-stride): UNR entries' index and value loads issued before their
// gathers; the x store per row. How much memory-level parallelism per thread
// does the 27-point SpMV need?
template <int UNR, bool STREAM>
__global__ void __launch_bounds__(256) k_ell_like(const int* __restrict__ ci, const double* __restrict__ v,
                                                  const double* __restrict__ b, double* __restrict__ x, int64_t rows) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0;
#pragma unroll 1
        for (int k0 = 0; k0 < 27; k0 += UNR) {
            int c[UNR];
            double vv[UNR], g[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                c[u] = STREAM ? __ldcs(ci + (int64_t)(k0 + u) * rows + r) : __ldg(ci + (int64_t)(k0 + u) * rows + r);
                vv[u] = STREAM ? __ldcs(v + (int64_t)(k0 + u) * rows + r) : __ldg(v + (int64_t)(k0 + u) * rows + r);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) g[u] = __ldg(b + c[u]);
#pragma unroll
            for (int u = 0; u < UNR; ++u) acc += vv[u] * g[u];
        }
        x[r] = acc;
    }
}

// random gathers (C3-like): per entry one coalesced int32 column index, one
// 8-byte gather from a 33.5 MB vector (L2-resident), VEC entries per lane
template <int VEC>
__global__ void __launch_bounds__(256) k_rand_gather(const int* __restrict__ ci, const double* __restrict__ b,
                                                     int64_t n, double* out) {
    double s = 0;
    const int64_t nv = n / VEC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        int c[VEC];
        if (VEC == 4) {
            const int4 q = __ldcs(reinterpret_cast<const int4*>(ci) + i);
            c[0] = q.x; c[VEC > 1 ? 1 : 0] = q.y; c[VEC > 2 ? 2 : 0] = q.z; c[VEC > 3 ? 3 : 0] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < VEC; ++u) c[u] = __ldcs(ci + i * VEC + u);
        }
#pragma unroll
        for (int u = 0; u < VEC; ++u) s += __ldg(b + c[u]);
    }
    if (s == 12345.678) *out = s;
}

template <typename F>
static float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}

int main() {
    const int64_t bytes = 1ll << 30, n2 = bytes / 16;
    double2* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per_sm : {4, 8}) {
        const int grid = sms * per_sm;
        float ms = timeit([&] { k_gridstride<<<grid, 256>>>(a, n2); });
        printf("gridstride   grid %5d             : %7.1f GB/s\n", grid, bytes / ms / 1e6);
    }
    for (int64_t chunk : {16384ll, 65536ll, 196608ll, 786432ll}) {
        const int64_t per = chunk / 16;
        const int64_t grid = (n2 + per - 1) / per;
        float ms = timeit([&] { k_chunk_cta<<<(unsigned)grid, 256>>>(a, n2, per); });
        printf("chunk/CTA    chunk %7lld B        : %7.1f GB/s\n", (long long)chunk, bytes / ms / 1e6);
    }
    for (int64_t chunk : {4096ll, 16384ll, 65536ll}) {
        const int64_t per = chunk / 16;
        const int64_t warps = (n2 + per - 1) / per;
        float ms = timeit([&] { k_chunk_warp<<<(unsigned)((warps + 7) / 8), 256>>>(a, n2, per); });
        printf("chunk/warp   chunk %7lld B        : %7.1f GB/s\n", (long long)chunk, bytes / ms / 1e6);
    }
    const int grid = sms * 8;
    const char* pol[] = {"ldcs", "ldg", "plain"};
#define WIDTH(T, P)                                                                                     \
    {                                                                                                   \
        float ms = timeit([&] { k_width<T, P><<<grid, 256>>>((const T*)a, bytes / (int64_t)sizeof(T)); }); \
        printf("gridstride %2d-byte loads, %-5s   : %7.1f GB/s\n", (int)sizeof(T), pol[P], bytes / ms / 1e6); \
    }
    WIDTH(float, 0) WIDTH(float, 1) WIDTH(float, 2)
    WIDTH(double, 0) WIDTH(double, 1) WIDTH(double, 2)
    WIDTH(double2, 0) WIDTH(double2, 1) WIDTH(double2, 2)
    {
        // 56.6M entries (C2), 27-point-like columns over 2.1M rows
        const int64_t n = 56623104, rows = 2097152;
        int* ci;
        double *v, *bb, *x;
        cudaMalloc(&ci, n * 4);
        cudaMalloc(&v, n * 8);
        cudaMalloc(&bb, rows * 8);
        cudaMalloc(&x, rows * 8);
        cudaMemset(bb, 0, rows * 8);
        cudaMemset(v, 0, n * 8);
        int* h = (int*)malloc(n * 4);
        const int off[27] = {-16513, -16512, -16511, -16385, -16384, -16383, -16257, -16256, -16255,
                             -129, -128, -127, -1, 0, 1, 127, 128, 129,
                             16255, 16256, 16257, 16383, 16384, 16385, 16511, 16512, 16513};
        for (int64_t k = 0; k < n; ++k) {
            int64_t c = k / 27 + off[k % 27];
            h[k] = (int)(c < 0 ? 0 : c >= rows ? rows - 1 : c);
        }
        cudaMemcpy(ci, h, n * 4, cudaMemcpyHostToDevice);
        free(h);
        const double by = n * 12.0, byw = by + rows * 8.0;
#define SPL(VEC, G, W)                                                                                    \
        {                                                                                                 \
            float ms = timeit([&] { k_spmv_like<VEC, G, W><<<grid, 256>>>(ci, v, bb, x, n); });           \
            printf("spmv-like vec %d gather %d write %d       : %7.1f GB/s (matrix%s bytes)\n", VEC, G, W, \
                   (W ? byw : by) / ms / 1e6, W ? " + x" : "");                                           \
        }
        SPL(1, false, false) SPL(4, false, false) SPL(1, true, false) SPL(4, true, false)
        SPL(1, false, true) SPL(4, false, true) SPL(1, true, true) SPL(4, true, true)
        // column-major copy of the same columns for the Ell-like kernels
        {
            int* hc = (int*)malloc(n * 4);
            int* hr = (int*)malloc(n * 4);
            cudaMemcpy(hr, ci, n * 4, cudaMemcpyDeviceToHost);
            for (int64_t r = 0; r < rows; ++r)
                for (int k = 0; k < 27; ++k) hc[(int64_t)k * rows + r] = hr[r * 27 + k];
            cudaMemcpy(ci, hc, n * 4, cudaMemcpyHostToDevice);
            free(hc);
            free(hr);
        }
        const double bye = n * 12.0 + rows * 16.0;  // matrix + b + x
#define ELL(UNR, ST, PER_SM)                                                                                  \
        {                                                                                                     \
            float ms = timeit([&] { k_ell_like<UNR, ST><<<sms * PER_SM, 256>>>(ci, v, bb, x, rows); });         \
            printf("ell-like unroll %2d %s per_sm %2d        : %7.1f GB/s (matrix + b + x)\n", UNR,            \
                   ST ? "ldcs" : "ldg ", PER_SM, bye / ms / 1e6);                                             \
        }
        ELL(1, false, 8) ELL(3, false, 8) ELL(9, false, 8) ELL(27, false, 8)
        ELL(3, true, 8) ELL(9, true, 8) ELL(27, true, 8)
        ELL(9, false, 4) ELL(9, false, 16) ELL(27, false, 4)
    }
    {
        // C3-like: 67.1M random columns over 4,194,304 rows
        const int64_t n = 67108864, cols = 4194304;
        int* ci;
        double *bb, *o;
        cudaMalloc(&ci, n * 4);
        cudaMalloc(&bb, cols * 8);
        cudaMalloc(&o, 8);
        cudaMemset(bb, 0, cols * 8);
        int* h = (int*)malloc(n * 4);
        unsigned long long st = 88172645463325252ull;
        for (int64_t k = 0; k < n; ++k) {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            h[k] = (int)(st % cols);
        }
        cudaMemcpy(ci, h, n * 4, cudaMemcpyHostToDevice);
        free(h);
        for (int per_sm : {4, 8, 16}) {
            float ms = timeit([&] { k_rand_gather<1><<<sms * per_sm, 256>>>(ci, bb, n, o); });
            printf("random gather vec 1 per_sm %2d   : %7.1f us  %6.1f G gathers/s\n", per_sm, ms * 1e3, n / ms / 1e6);
            ms = timeit([&] { k_rand_gather<4><<<sms * per_sm, 256>>>(ci, bb, n, o); });
            printf("random gather vec 4 per_sm %2d   : %7.1f us  %6.1f G gathers/s\n", per_sm, ms * 1e3, n / ms / 1e6);
        }
    }
    return 0;
}
