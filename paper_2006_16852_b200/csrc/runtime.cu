// C-ABI runtime: error strings, launch accounting, prefix scans, reductions
// and the BLAS-1 kernels behind Dense (reference src/formats.py:121-147 ->
// src/kernels.py:30-137: Copy/Fill/Scale/AddScaled/Dot/Norm2).
//
// Dense vectors are row-major (n, m) with a row stride (src/formats.py:70-86);
// per-column scalars are (1, m) device arrays or one host value.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>

#include "common.cuh"

namespace b200sp {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};
static thread_local const int* g_guard = nullptr;

const int* current_guard() { return g_guard; }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
        return B200SP_ECUDA;
    }
    return B200SP_OK;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Tuning knobs (kernel variants / launch shapes) for sweeps; every knob has
// the measured-best default at its call site (tuning(key, default)).
static constexpr int kMaxKnobs = 32;
static char g_knob_key[kMaxKnobs][32];
static int g_knob_val[kMaxKnobs];
static std::atomic<int> g_knobs{0};

int tuning(const char* key, int dflt) {
    const int k = g_knobs.load(std::memory_order_acquire);
    for (int i = 0; i < k; ++i)
        if (std::strncmp(g_knob_key[i], key, sizeof(g_knob_key[i])) == 0)
            return g_knob_val[i] == B200SP_TUNING_DEFAULT ? dflt : g_knob_val[i];
    return dflt;
}

// ---------------------------------------------------------------------------
// exclusive scan (int32 in -> int32/int64 out, with total at out[count])
// three phases: tile sums, single-CTA scan of tile sums, tile scan + offset
// ---------------------------------------------------------------------------
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_IPT;

__global__ void scan_tile_sums(int64_t count, const int* __restrict__ in, long long* __restrict__ sums) {
    __shared__ long long sh[SCAN_BLOCK / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    long long s = 0;
    for (int i = threadIdx.x; i < SCAN_TILE; i += SCAN_BLOCK) {
        int64_t k = base + i;
        if (k < count) s += in[k];
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void scan_sums_single(int64_t nt, long long* __restrict__ sums) {
    // one CTA of 1024 threads, chunks of 1024 with running carry
    __shared__ long long sh[1024];
    long long carry = 0;
    for (int64_t base = 0; base < nt; base += 1024) {
        int64_t k = base + threadIdx.x;
        long long v = k < nt ? sums[k] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            long long t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (k < nt) sums[k] = carry + sh[threadIdx.x] - v;  // exclusive
        long long tot = sh[1023];
        __syncthreads();
        carry += tot;
    }
}

template <typename OUT>
__global__ void scan_tiles(int64_t count, const int* __restrict__ in, const long long* __restrict__ offs,
                           OUT* __restrict__ out) {
    __shared__ long long wsum[SCAN_BLOCK / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    long long loc[SCAN_IPT];
    long long t = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        int64_t k = base + i;
        loc[i] = k < count ? in[k] : 0;
        t += loc[i];
    }
    // warp inclusive scan of thread totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long n2 = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n2;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    long long wpre = 0;
    for (int w = 0; w < wid; ++w) wpre += wsum[w];
    long long run = offs[blockIdx.x] + wpre + incl - t;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        int64_t k = base + i;
        if (k < count) out[k] = (OUT)run;
        run += loc[i];
    }
    if (base <= count - 1 && count - 1 < base + SCAN_IPT) out[count] = (OUT)run;  // total
}

template <typename OUT>
static int exclusive_scan(int64_t count, const int* in, OUT* out, long long* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (count == 0) {
        B200SP_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(OUT), st));
        return B200SP_OK;
    }
    const int64_t nt = ceil_div(count, SCAN_TILE);
    scan_tile_sums<<<(unsigned)nt, SCAN_BLOCK, 0, st>>>(count, in, ws);
    scan_sums_single<<<1, 1024, 0, st>>>(nt, ws);
    scan_tiles<OUT><<<(unsigned)nt, SCAN_BLOCK, 0, st>>>(count, in, ws, out);
    count_launch(3);
    return check_launch("exclusive_scan");
}

// ---------------------------------------------------------------------------
// int reductions (max / sum) into a device scalar
// ---------------------------------------------------------------------------
__global__ void reduce_max_i32_kernel(int64_t count, const int* __restrict__ in, int* __restrict__ out) {
    int m = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, in[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ---------------------------------------------------------------------------
// BLAS-1 on (n, m) row-major dense blocks
// ---------------------------------------------------------------------------
template <typename T>
__global__ void fill_kernel(int64_t n, int m, T* __restrict__ x, int64_t xs, T value) {
    const int64_t tot = n * m;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / m, j = t - i * m;
        x[i * xs + j] = value;
    }
}

template <typename T>
__global__ void copy_kernel(int64_t n, int m, const T* __restrict__ s, int64_t ss, T* __restrict__ d, int64_t ds) {
    const int64_t tot = n * m;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / m, j = t - i * m;
        d[i * ds + j] = s[i * ss + j];
    }
}

// x <- alpha * x ; alpha per column (alpha_dev[j]) or one host value
template <typename T>
__global__ void scale_kernel(int64_t n, int m, T alpha, const T* __restrict__ alpha_dev, T* __restrict__ x, int64_t xs) {
    const int64_t tot = n * m;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / m, j = t - i * m;
        const T a = alpha_dev ? alpha_dev[j] : alpha;
        x[i * xs + j] = x[i * xs + j] * a;
    }
}

// y <- y + alpha * x
template <typename T>
__global__ void add_scaled_kernel(int64_t n, int m, T alpha, const T* __restrict__ alpha_dev,
                                  const T* __restrict__ x, int64_t xs, T* __restrict__ y, int64_t ys) {
    const int64_t tot = n * m;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / m, j = t - i * m;
        const T a = alpha_dev ? alpha_dev[j] : alpha;
        // product rounded before the add (no FMA contraction): the same two
        // roundings as the reference's NumPy `y + a * x` (src/kernels.py:94-110)
        y[i * ys + j] = y[i * ys + j] + mul_rn(a, x[i * xs + j]);
    }
}

// Deterministic two-level dot / squared-norm: a fixed grid writes per-block
// partials, the last CTA to finish (ticket counter) sums them in block order.
constexpr int RED_BLOCK = 256;
constexpr int RED_MAX_COLS = 64;

template <typename T, bool NORM>
__global__ void __launch_bounds__(RED_BLOCK)
dot_kernel(int64_t n, int m, const T* __restrict__ x, int64_t xs, const T* __restrict__ y, int64_t ys,
           T* __restrict__ out, T* __restrict__ partials, unsigned* __restrict__ counter) {
    __shared__ T sh[RED_BLOCK / 32];
    __shared__ bool last;
    for (int j = 0; j < m; ++j) {
        T s = 0;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            const T a = x[i * xs + j];
            s += a * (NORM ? a : y[i * ys + j]);
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) partials[(int64_t)blockIdx.x * m + j] = s;
    }
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int j = 0; j < m; ++j) {
        T s = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += partials[(int64_t)b * m + j];
        s = block_sum(s, sh);
        if (threadIdx.x == 0) out[j] = NORM ? sqrt(s) : s;
    }
    if (threadIdx.x == 0) *counter = 0;
}

template <typename T, bool NORM>
static int dot_impl(int64_t n, int m, const T* x, int64_t xs, const T* y, int64_t ys, T* out,
                    T* partials, unsigned* counter, void* stream) {
    B200SP_REQUIRE(m >= 1 && m <= RED_MAX_COLS, B200SP_EINVAL, "dot: 1 <= m <= %d", RED_MAX_COLS);
    cudaStream_t st = as_stream(stream);
    const int grid = grid_for(n, RED_BLOCK, 4);
    dot_kernel<T, NORM><<<grid, RED_BLOCK, 0, st>>>(n, m, x, xs, y, ys, out, partials, counter);
    count_launch();
    return check_launch(NORM ? "norm2" : "dot");
}

}  // namespace b200sp

using namespace b200sp;

extern "C" {

const char* b200sp_last_error(void) { return g_err; }
long long b200sp_launch_count(void) { return g_launches.load(); }
int b200sp_version(void) { return B200SP_ABI_VERSION; }
void b200sp_set_guard(const int32_t* guard) { g_guard = guard; }

int b200sp_set_tuning(const char* key, int32_t value) {
    const int k = g_knobs.load(std::memory_order_acquire);
    for (int i = 0; i < k; ++i)
        if (std::strncmp(g_knob_key[i], key, sizeof(g_knob_key[i])) == 0) {
            g_knob_val[i] = value;
            return B200SP_OK;
        }
    B200SP_REQUIRE(k < kMaxKnobs, B200SP_EINVAL, "set_tuning: too many knobs");
    B200SP_REQUIRE(std::strlen(key) < sizeof(g_knob_key[0]), B200SP_EINVAL, "set_tuning: key too long");
    std::strncpy(g_knob_key[k], key, sizeof(g_knob_key[k]));
    g_knob_val[k] = value;
    g_knobs.store(k + 1, std::memory_order_release);
    return B200SP_OK;
}
int64_t b200sp_reduce_workspace_elems(void) { return (int64_t)kNumSMs * 4 * RED_MAX_COLS; }

int b200sp_device_sync(void) {
    B200SP_CHECK_CUDA(cudaDeviceSynchronize());
    return B200SP_OK;
}

int64_t b200sp_scan_workspace_elems(int64_t count) { return ceil_div(count, SCAN_TILE) + 1; }

int b200sp_exclusive_scan_i32(int64_t count, const int32_t* in, int32_t* out, long long* ws, void* stream) {
    return exclusive_scan<int>(count, in, out, ws, stream);
}
int b200sp_exclusive_scan_i64(int64_t count, const int32_t* in, int64_t* out, long long* ws, void* stream) {
    return exclusive_scan<long long>(count, in, (long long*)out, ws, stream);
}

int b200sp_reduce_max_i32(int64_t count, const int32_t* in, int32_t* out, void* stream) {
    cudaStream_t st = as_stream(stream);
    B200SP_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(int), st));  // lengths are >= 0
    if (count == 0) return B200SP_OK;
    reduce_max_i32_kernel<<<grid_for(count, 256, 4), 256, 0, st>>>(count, in, out);
    count_launch();
    return check_launch("reduce_max_i32");
}

#define BLAS1(T, SUF)                                                                                 \
    int b200sp_fill_##SUF(int64_t n, int32_t m, T* x, int64_t xs, T value, void* stream) {            \
        if (n * m == 0) return B200SP_OK;                                                             \
        fill_kernel<T><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, x, xs, value);   \
        count_launch();                                                                               \
        return check_launch("fill");                                                                  \
    }                                                                                                 \
    int b200sp_copy_##SUF(int64_t n, int32_t m, const T* s, int64_t ss, T* d, int64_t ds, void* stream) { \
        if (n * m == 0) return B200SP_OK;                                                             \
        copy_kernel<T><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, s, ss, d, ds);   \
        count_launch();                                                                               \
        return check_launch("copy");                                                                  \
    }                                                                                                 \
    int b200sp_scale_##SUF(int64_t n, int32_t m, T alpha, const T* alpha_dev, T* x, int64_t xs,       \
                           void* stream) {                                                            \
        if (n * m == 0) return B200SP_OK;                                                             \
        scale_kernel<T><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, alpha, alpha_dev, x, xs); \
        count_launch();                                                                               \
        return check_launch("scale");                                                                 \
    }                                                                                                 \
    int b200sp_add_scaled_##SUF(int64_t n, int32_t m, T alpha, const T* alpha_dev, const T* x,       \
                                int64_t xs, T* y, int64_t ys, void* stream) {                         \
        if (n * m == 0) return B200SP_OK;                                                             \
        add_scaled_kernel<T><<<grid_for(n * m, 256, 8), 256, 0, as_stream(stream)>>>(n, m, alpha, alpha_dev, x, xs, y, ys); \
        count_launch();                                                                               \
        return check_launch("add_scaled");                                                            \
    }                                                                                                 \
    int b200sp_dot_##SUF(int64_t n, int32_t m, const T* x, int64_t xs, const T* y, int64_t ys, T* out, \
                         T* partials, uint32_t* counter, void* stream) {                              \
        return dot_impl<T, false>(n, m, x, xs, y, ys, out, partials, counter, stream);                \
    }                                                                                                 \
    int b200sp_norm2_##SUF(int64_t n, int32_t m, const T* x, int64_t xs, T* out, T* partials,        \
                           uint32_t* counter, void* stream) {                                         \
        return dot_impl<T, true>(n, m, x, xs, x, xs, out, partials, counter, stream);                 \
    }

BLAS1(double, f64)
BLAS1(float, f32)

}  // extern "C"
